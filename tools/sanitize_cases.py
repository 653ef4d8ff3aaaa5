"""Small launches of every kernel kind, for compute-sanitizer (memcheck,
racecheck, synccheck, initcheck): every fused family (halo-staged direct,
row-segment and its warp-specialised TMA variant, 16-byte, 4-byte and
persistent warp-specialised pointwise), split-C through partial planes + stage 2 and
through DSMEM clusters, the paper-faithful stage 1 + stage 2, and the tcgen05
engines in halo and gather mode (3xTF32 with bf16 corrections, TF32).
Each result is checked against the oracle so a sanitizer run is also a
numerics run.   python tools/sanitize_cases.py [--quick]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2103_16234_b200 as pk  # noqa: E402

CASES = [
    pk.ConvConfig("3x3", n=2, c=24, h=14, w=14, m=40, hf=3, wf=3, pad_h=1, pad_w=1),
    pk.ConvConfig("1x1v", n=2, c=64, h=14, w=14, m=48, hf=1, wf=1),
    pk.ConvConfig("1x1t", n=3, c=48, h=16, w=16, m=72, hf=1, wf=1),
    pk.ConvConfig("1x1img", n=7, c=48, h=7, w=7, m=80, hf=1, wf=1),
    pk.ConvConfig("1x1odd", n=3, c=40, h=7, w=7, m=36, hf=1, wf=1),
    pk.ConvConfig("1x1s2", n=2, c=32, h=14, w=14, m=40, hf=1, wf=1, stride=2),
    pk.ConvConfig("5x5", n=1, c=16, h=14, w=14, m=32, hf=5, wf=5, pad_h=2, pad_w=2),
    pk.ConvConfig("7x7s2", n=1, c=3, h=32, w=32, m=16, hf=7, wf=7, stride=2, pad_h=3, pad_w=3),
    pk.ConvConfig("3x3s2", n=2, c=16, h=15, w=15, m=24, hf=3, wf=3, stride=2, pad_h=1, pad_w=1),
    pk.ConvConfig("gen", n=1, c=8, h=9, w=7, m=5, hf=2, wf=4, stride=3, pad_h=1, pad_w=2),
]


def main():
    quick = "--quick" in sys.argv
    torch.cuda.set_device(0)
    n = 0
    for i, cfg in enumerate(CASES):
        xn = oracle.make_uniform(pk.input_dims(cfg), 10 + i)
        wn = oracle.make_uniform(pk.filter_dims(cfg), 20 + i)
        x, w = torch.from_numpy(xn).cuda(), torch.from_numpy(wn).cuda()
        ref = oracle.conv_f64(cfg, xn, wn)
        tol = oracle.fp32_tolerance(cfg.c, cfg.hf, cfg.wf)
        fams = pk.matching_families(cfg)
        if quick:  # two round-1 families plus every row-segment / warp-specialised one
            names = pk.family_names()
            fams = fams[:2] + [f for f in fams[2:] if any(k in names[f] for k in ("row7", "rws7", "1x1ws", "1x1t_", "1x1pk"))]
        for fam in fams:
            for splits, reduce in ((1, 0), (2, 1), (2, 2)):
                try:
                    layer = pk.ConvLayer(cfg, family=fam, splits=splits, reduce=reduce)
                except pk.InvalidPlan:
                    continue
                y = layer(x, w)
                torch.cuda.synchronize()
                err = oracle.relative_error(y.cpu().numpy(), ref)
                assert err <= tol, (cfg.name, layer.family, splits, reduce, err)
                n += 1
        for engine in ("tf32x3", "tf32"):
            y = pk.ConvLayer(cfg, engine)(x, w)
            torch.cuda.synchronize()
            err = oracle.relative_error(y.cpu().numpy(), ref)
            assert err <= (tol if engine == "tf32x3" else 5e-3), (cfg.name, engine, err)
            n += 1
        if cfg.stride == 1:
            out, _ = pk.conv_twostage(pk.Tensor4(xn), pk.Tensor4(wn), cfg)
            assert out.data.tobytes() == oracle.conv_naive(cfg, xn, wn).tobytes(), cfg.name
            n += 1
    print(f"sanitize cases ok: {n} launches checked")


if __name__ == "__main__":
    main()
