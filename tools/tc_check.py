"""Development check of the tensor-core engines on the GPU box (not a test).

    python tools/tc_check.py            # numerics on small/edge shapes + timings on BASELINE layers
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

from paper_2103_16234_b200 import ConvConfig, ConvLayer
from paper_2103_16234_b200 import workloads as W


def rel(a, b):
    return float((a.double() - b).abs().max() / b.abs().max())


def trunc_tf32(t):
    return (t.view(torch.int32) & -8192).view(torch.float32)


def rn_tf32(t):
    i = t.view(torch.int32).to(torch.int64)
    i = (i + 0x1000 + ((i >> 13) & 1) - 1) & ~0x1FFF  # round half to even on the 13 dropped bits
    return i.to(torch.int32).view(torch.float32)


def case(name, n, c, h, w, m, f, pad, stride=1, engines=("tf32x3", "tf32")):
    cfg = ConvConfig(name, n=n, c=c, h=h, w=w, m=m, hf=f, wf=f, stride=stride, pad_h=pad, pad_w=pad)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.rand((n, c, h, w), device="cuda", generator=g) * 2 - 1
    wt = torch.rand((m, c, f, f), device="cuda", generator=g) * 2 - 1
    ref = F.conv2d(x.double(), wt.double(), padding=pad, stride=stride)
    out = {"case": name}
    for e in engines:
        try:
            L = ConvLayer(cfg, e)
            y = L(x, wt)
            torch.cuda.synchronize()
            out[e] = rel(y, ref)
            out[e + "_plan"] = L.family
            if e == "tf32":
                out["tf32_vs_trunc_model"] = rel(y, F.conv2d(trunc_tf32(x).double(), trunc_tf32(wt).double(), padding=pad,
                                                              stride=stride))
        except Exception as ex:  # noqa: BLE001
            out[e] = f"ERR {type(ex).__name__}: {ex}"[:300]
    print(json.dumps(out), flush=True)


def timing(wl, n, names=None, reps=20):
    rows = []
    for cfg in W.layers(wl, n):
        if names and cfg.name not in names:
            continue
        x = torch.rand((cfg.n, cfg.c, cfg.h, cfg.w), device="cuda") * 2 - 1
        wt = torch.rand((cfg.m, cfg.c, cfg.hf, cfg.wf), device="cuda") * 2 - 1
        r = {"layer": cfg.name, "n": n}
        for e in ("fused", "tf32x3", "tf32"):
            try:
                L = ConvLayer(cfg, e)
            except Exception as ex:  # noqa: BLE001
                r[e] = "unsupported"
                continue
            y = L(x, wt)
            for _ in range(3):
                L(x, wt, out=y)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                L(x, wt, out=y)
            b.record()
            b.synchronize()
            us = a.elapsed_time(b) / reps * 1e3
            r[e] = round(us, 2)
            r[e + "_tf"] = round(cfg.flops / us / 1e6, 1)
            r[e + "_plan"] = L.family
        print(json.dumps(r), flush=True)
        rows.append(r)
    return rows


CASES = {
    "1x1-tiny": (1, 16, 4, 8, 16, 1, 0), "1x1-a": (2, 64, 8, 8, 64, 1, 0), "1x1-flat196": (3, 48, 14, 14, 40, 1, 0),
    "1x1-M300": (2, 96, 28, 28, 300, 1, 0), "1x1-C5": (1, 5, 8, 8, 24, 1, 0), "1x1-deepK": (2, 256, 8, 8, 64, 1, 0),
    "1x1-pad-w32": (1, 16, 30, 32, 16, 1, 1), "1x1-pad-w16": (1, 16, 14, 16, 16, 1, 1),
    "3x3-w32": (1, 16, 8, 32, 16, 3, 1), "3x3-w32-nopad": (1, 16, 8, 32, 16, 3, 0), "3x3-w16": (1, 16, 16, 16, 16, 3, 1),
    "3x3-a": (2, 32, 16, 16, 64, 3, 1), "3x3-w28": (2, 64, 28, 28, 128, 3, 1), "3x3-w56": (1, 64, 56, 56, 64, 3, 1),
    "3x3-c3": (2, 3, 32, 32, 64, 3, 1), "5x5-w28": (2, 32, 28, 28, 96, 5, 2), "3x3-nopad": (2, 40, 12, 12, 48, 3, 0),
    "3x3-w224": (1, 16, 224, 224, 64, 3, 1), "3x3-w7": (4, 64, 7, 7, 80, 3, 1), "5x5-w27": (2, 24, 27, 27, 40, 5, 2),
    "3x3-s2": (2, 32, 15, 15, 48, 3, 1, 2), "1x1-s2": (2, 64, 14, 14, 96, 1, 0, 2), "7x7-s2": (1, 3, 40, 40, 64, 7, 3, 2),
    "even-2x4": (2, 8, 9, 10, 24, 2, 1), "1x1-w49": (8, 832, 7, 7, 48, 1, 0),
}

if __name__ == "__main__":
    import subprocess
    if len(sys.argv) > 2 and sys.argv[1] == "time":  # time WL N name,name,...
        torch.cuda.set_device(0)
        for spec in sys.argv[2:]:
            wl, n, names = spec.split(":")
            timing(wl, int(n), names=set(names.split(",")) if names else None)
        sys.exit(0)
    if len(sys.argv) > 2 and sys.argv[1] == "case":
        torch.cuda.set_device(0)
        case(sys.argv[2], *CASES[sys.argv[2]])
        sys.exit(0)
    for name in CASES:
        r = subprocess.run([sys.executable, __file__, "case", name], capture_output=True, text=True, timeout=120)
        print(r.stdout.strip() or f'{{"case": "{name}", "rc": {r.returncode}, "err": {json.dumps(r.stderr[-300:])}}}',
              flush=True)
    if "--quick" in sys.argv:
        sys.exit(0)
    torch.cuda.set_device(0)
    timing("c1", 1)
    timing("c2", 32)
    timing("c3", 128)
    timing("c4", 8)
    timing("c5", 256, names={"layer1.0.conv2", "layer2.1.conv2", "layer3.1.conv2", "layer1.0.conv3", "layer3.1.conv1"})


def _unused():
    case("1x1-tiny", 1, 16, 4, 8, 16, 1, 0)
    case("1x1-a", 2, 64, 8, 8, 64, 1, 0)
    case("1x1-flat196", 3, 48, 14, 14, 40, 1, 0)
    case("1x1-M300", 2, 96, 28, 28, 300, 1, 0)
    case("1x1-C5", 1, 5, 8, 8, 24, 1, 0)
    case("3x3-a", 2, 32, 16, 16, 64, 3, 1)
    case("3x3-w28", 2, 64, 28, 28, 128, 3, 1)
    case("3x3-w56", 1, 64, 56, 56, 64, 3, 1)
    case("3x3-c3", 2, 3, 32, 32, 64, 3, 1)
    case("5x5-w28", 2, 32, 28, 28, 96, 5, 2)
    case("3x3-nopad", 2, 40, 12, 12, 48, 3, 0)
    case("3x3-w224", 1, 16, 224, 224, 64, 3, 1)
    if "--quick" in sys.argv:
        sys.exit(0)
    timing("c1", 1)
    timing("c2", 32)
    timing("c3", 128)
    timing("c4", 8)
    timing("c5", 256, names={"layer1.0.conv2", "layer2.1.conv2", "layer3.1.conv2", "layer1.0.conv3", "layer3.1.conv1"})
