"""Generate the golden fixtures that pin the oracle (and, through it, the
CUDA engine) to the reference implementation.

Run in the build container, where the reference is importable:

    python tests/golden/make_golden.py            # writes tests/golden/*.json|npz

It imports convkit from $CONVKIT_REF or /root/reference/pkg/src and records,
for seeded inputs drawn exactly as the reference draws them
(tensor.make_tensor, tensor.py:80-109; harness seeds, bench.py:119-121):

* sha256 of conv_naive / conv_twostage / conv_naive_f64 outputs
  (reference.py:58-103, twostage.py:208-239) on
  - the acceptance corpus (seed 2024, 200 configs; test_acceptance.py:38-59),
  - a stride/asymmetric-pad/even-filter corpus (conv_naive handles any stride),
  - the 7 presets with seeds 1000+i / 2000+i (test_acceptance.py:62-71),
  - BASELINE.md layers at small N with the harness seeds;
* RunStats, workspace_bytes and plan_launch for the presets and a plan corpus
  (twostage.py:36-55, execmodel.py:73-98);
* full arrays for small special-value cases (NaN/Inf/-0.0/denormals), where
  the reference's separate-rounding semantics are most fragile.

Nothing at test time reads /root/reference: tests consume only these files.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("CONVKIT_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import convkit as ck  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float32).tobytes()).hexdigest()


def cfg_dict(cfg):
    return {k: getattr(cfg, k) for k in ("name", "n", "c", "h", "w", "m", "hf", "wf", "stride", "pad_h", "pad_w")}


def run_case(cfg, seed_in, seed_f, *, twostage=True, f64=True):
    x = ck.make_tensor(ck.input_dims(cfg), "uniform", seed=seed_in)
    w = ck.make_tensor(ck.filter_dims(cfg), "uniform", seed=seed_f)
    rec = {"cfg": cfg_dict(cfg), "seed_in": seed_in, "seed_f": seed_f,
           "naive": sha(ck.conv_naive(x, w, cfg).data)}
    if twostage and cfg.stride == 1:
        out, stats = ck.conv_twostage(x, w, cfg, workspace_limit=1 << 62)
        rec["twostage"] = sha(out.data)
        rec["stats"] = {"stage1_tasks_run": stats.stage1_tasks_run, "stage2_invoked": stats.stage2_invoked,
                        "filter_row_global_loads": stats.filter_row_global_loads,
                        "workspace_bytes": stats.workspace_bytes}
    if f64:
        rec["f64"] = sha(ck.conv_naive_f64(x, w, cfg).data)
    return rec


def corpus_2024():
    # same draw sequence as test_acceptance._random_corpus(seed=2024, count=200)
    rng = np.random.default_rng(2024)
    cases = []
    for i in range(200):
        f = int(rng.choice((1, 3, 5)))
        ph, pw = ck.same_padding(f, f)
        cfg = ck.ConvConfig(f"r{i}", n=int(rng.integers(1, 5)), c=int(rng.integers(1, 65)),
                            h=int(rng.integers(1, 33)), w=int(rng.integers(1, 33)),
                            m=int(rng.integers(1, 33)), hf=f, wf=f, pad_h=ph, pad_w=pw)
        si, sf = int(rng.integers(1 << 31)), int(rng.integers(1 << 31))
        cases.append(run_case(cfg, si, sf))
    return cases


def corpus_general():
    # any stride / asymmetric pads / even and rectangular filters / odd planes
    rng = np.random.default_rng(7007)
    cases = []
    while len(cases) < 80:
        hf, wf = int(rng.integers(1, 8)), int(rng.integers(1, 8))
        s = int(rng.choice((1, 1, 2, 2, 3)))
        ph, pw = int(rng.integers(0, 4)), int(rng.integers(0, 4))
        h, w = int(rng.integers(1, 30)), int(rng.integers(1, 30))
        if hf > h + 2 * ph or wf > w + 2 * pw:
            continue
        cfg = ck.ConvConfig(f"g{len(cases)}", n=int(rng.integers(1, 4)), c=int(rng.integers(1, 40)),
                            h=h, w=w, m=int(rng.integers(1, 24)), hf=hf, wf=wf, stride=s, pad_h=ph, pad_w=pw)
        cases.append(run_case(cfg, int(rng.integers(1 << 31)), int(rng.integers(1 << 31))))
    return cases


def presets():
    recs = []
    for i, cfg in enumerate(ck.preset_configs()):
        r = run_case(cfg, 1000 + i, 2000 + i)
        p = ck.plan_launch(cfg)
        r["plan"] = [p.blocks, p.threads_per_block, p.split_per_filter_row, p.dot_products_per_thread]
        r["workspace_bytes"] = ck.workspace_bytes(cfg)
        recs.append(r)
    return recs


# BASELINE.md layer shapes: (name, c, h, m, f, stride, pad)
BASELINE_LAYERS = [
    ("res-conv2x-3x3", 64, 56, 64, 3, 1, 1),
    ("3a-1x1", 192, 28, 64, 1, 1, 0), ("3a-5x5red", 192, 28, 16, 1, 1, 0),
    ("4a-1x1", 480, 14, 192, 1, 1, 0), ("4e-1x1", 528, 14, 256, 1, 1, 0),
    ("5a-5x5red", 832, 7, 32, 1, 1, 0), ("5b-1x1", 832, 7, 384, 1, 1, 0),
    ("alexnet-conv2", 96, 27, 256, 5, 1, 2), ("incep-3b-5x5", 32, 28, 96, 5, 1, 2),
    ("incep-5b-5x5", 48, 7, 128, 5, 1, 2),
    ("vgg1_1", 3, 224, 64, 3, 1, 1), ("vgg3_1", 128, 56, 256, 3, 1, 1), ("vgg5_1", 512, 14, 512, 3, 1, 1),
    ("conv1", 3, 224, 64, 7, 2, 3), ("layer2.0.conv2", 128, 56, 128, 3, 2, 1),
    ("layer2.0.downsample", 256, 56, 512, 1, 2, 0), ("layer4.1.conv2", 512, 7, 512, 3, 1, 1),
]


def baseline_layers():
    recs = []
    for idx, (name, c, h, m, f, s, p) in enumerate(BASELINE_LAYERS):
        for n in (1, 2):
            cfg = ck.ConvConfig(name, n=n, c=c, h=h, w=h, m=m, hf=f, wf=f, stride=s, pad_h=p, pad_w=p)
            si, sf = np.random.SeedSequence([0, idx, n]).generate_state(2)
            recs.append(run_case(cfg, int(si), int(sf), twostage=(n == 1)))
    return recs


def plan_corpus():
    rng = np.random.default_rng(99)
    recs = []
    for _ in range(300):
        f = int(rng.choice((1, 2, 3, 5, 7)))
        pad = int(rng.integers(0, 3))
        h = int(rng.integers(max(1, f - 2 * pad), 64))
        w = int(rng.integers(max(1, f - 2 * pad), 64))
        cfg = ck.ConvConfig("p", n=int(rng.integers(1, 300)), c=int(rng.integers(1, 9)), h=h, w=w,
                            m=int(rng.integers(1, 600)), hf=f, wf=f, pad_h=pad, pad_w=pad)
        dev = ck.DeviceModel(max_threads_per_block=int(rng.choice((1024, 512, 256, 1000, 100))))
        p = ck.plan_launch(cfg, dev)
        recs.append({"cfg": cfg_dict(cfg), "max_threads": dev.max_threads_per_block,
                     "plan": [p.blocks, p.threads_per_block, p.split_per_filter_row, p.dot_products_per_thread],
                     "workspace_bytes": ck.workspace_bytes(cfg)})
    return recs


def tensor_hashes():
    recs = []
    for seed, dims in ((5, (2, 256, 14, 14)), (0, (1, 1, 1, 1)), (123456789, (3, 7, 13, 27)), (2**31 - 1, (1, 64, 56, 56))):
        recs.append({"seed": seed, "dims": list(dims), "sha": sha(ck.make_tensor(dims, "uniform", seed=seed).data)})
    return recs


def special_values():
    """Small cases with NaN/Inf/-0.0/denormals: full reference outputs."""
    arrays = {}
    meta = []
    rng = np.random.default_rng(31)
    specials = np.array([np.nan, np.inf, -np.inf, -0.0, 0.0, 1e-40, -1e-42, 3.0e38, -3.0e38, 1.0], dtype=np.float32)
    for i in range(12):
        f = int(rng.choice((1, 3, 5)))
        p = int(rng.integers(0, (f + 1) // 2 + 1))
        cfg = ck.ConvConfig(f"sv{i}", n=int(rng.integers(1, 3)), c=int(rng.integers(1, 6)), h=int(rng.integers(f, 9)),
                            w=int(rng.integers(f, 9)), m=int(rng.integers(1, 4)), hf=f, wf=f, pad_h=p, pad_w=p)
        x = rng.uniform(-2, 2, ck.input_dims(cfg)).astype(np.float32)
        w = rng.uniform(-2, 2, ck.filter_dims(cfg)).astype(np.float32)
        kx = rng.random(x.shape) < 0.08
        kw = rng.random(w.shape) < (0.05 if i < 8 else 0.0)
        x[kx] = rng.choice(specials, size=int(kx.sum()))
        w[kw] = rng.choice(specials, size=int(kw.sum()))
        if i >= 8:  # denormal-heavy, finite
            x *= np.float32(1e-20); w *= np.float32(1e-19)
        out, _ = ck.conv_twostage(ck.Tensor4(x), ck.Tensor4(w), cfg)
        naive = ck.conv_naive(ck.Tensor4(x), ck.Tensor4(w), cfg).data
        assert out.data.tobytes() == naive.tobytes() or np.isnan(naive).any()
        arrays[f"sv{i}_x"], arrays[f"sv{i}_w"], arrays[f"sv{i}_naive"] = x, w, naive
        arrays[f"sv{i}_twostage"] = out.data
        meta.append(cfg_dict(cfg))
    return meta, arrays


def main():
    gold = {
        "generator": "tests/golden/make_golden.py",
        "reference": "convkit " + ck.__version__,
        "numpy": np.__version__,
        "tensor_hashes": tensor_hashes(),
        "presets": presets(),
        "corpus_2024": corpus_2024(),
        "corpus_general": corpus_general(),
        "baseline_layers": baseline_layers(),
        "plans": plan_corpus(),
    }
    meta, arrays = special_values()
    gold["special_values"] = meta
    (OUT / "golden.json").write_text(json.dumps(gold, indent=1))
    np.savez_compressed(OUT / "special_values.npz", **arrays)
    print(f"wrote {OUT/'golden.json'} and special_values.npz")


if __name__ == "__main__":
    main()
