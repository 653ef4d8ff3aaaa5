"""Development: dump CTA 0 of the tensor-core kernel (B2C_TC_DEBUG) and compare
with host expectations.  python tools/tc_debug.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

from paper_2103_16234_b200 import ConvConfig, ConvLayer

DUMP = "/tmp/tc_dump.bin"


def unswizzle(buf_bytes, L, swz):  # read logical byte offset L from a swizzled buffer
    bits = {128: 7, 64: 3}[swz]
    P = L ^ (((L >> 7) & bits) << 4)
    return buf_bytes[P:P + 4].view(np.float32)[0]


def run(name, n, c, h, w, m, f, pad, engine):
    os.environ["B2C_TC_DEBUG"] = DUMP
    cfg = ConvConfig(name, n=n, c=c, h=h, w=w, m=m, hf=f, wf=f, stride=1, pad_h=pad, pad_w=pad)
    torch.manual_seed(0)
    x = torch.rand((n, c, h, w), device="cuda") * 2 - 1
    wt = torch.rand((m, c, f, f), device="cuda") * 2 - 1
    L = ConvLayer(cfg, engine)
    print(name, engine, L.family, "grid", L.grid, flush=True)
    err = None
    try:
        y = L(x, wt)
        torch.cuda.synchronize()
    except Exception as ex:  # noqa: BLE001
        err = ex
    d = np.fromfile(DUMP, dtype=np.uint32)
    print("  code %#x cuda_err %d" % (d[0], d[1]), "exception:", err)
    if err is not None:
        return False
    st = d[16:16 + 65536].view(np.uint8)
    xs = x.cpu().numpy()
    ws = wt.cpu().numpy()
    xb = L._tc.pixels_per_chunk
    nf = L._tc.filters_per_tile
    # A tile of stage 0 (kb=0 -> tap 0, channels 0..15), flat 1x1 or rows mode
    bad = 0
    for ci in range(min(2, 128 // xb)):
        for cc in range(min(c, 16)):
            for xx in range(0, xb, 7):
                Lb = ci * xb * 64 + cc * xb * 4 + xx * 4
                got = unswizzle(st, Lb, xb * 4)
                if f == 1 and L._tc.flattened:
                    hw = ci * xb + xx
                    want = xs[0, cc].reshape(-1)[hw] if hw < h * w else 0.0
                else:
                    want = None
                if want is not None and got != want:
                    # tf32x3 splits hi in place: compare the hi part
                    hi = np.float32(np.uint32(np.float32(want).view(np.uint32) & 0xFFFFE000).view(np.float32))
                    if got != hi:
                        bad += 1
                        if bad < 5:
                            print(f"  A mismatch chunk {ci} c {cc} x {xx}: got {got} want {want}")
    print("  A-tile mismatches:", bad)
    bad = 0
    Boff = 8192
    for mm in range(min(nf, m)):
        for cc in range(min(c, 16)):
            got = unswizzle(st, Boff + mm * 64 + cc * 4, 64)
            want = ws[mm, cc, 0, 0] if f == 1 else None
            if want is not None and got != want:
                hi = np.float32(np.uint32(np.float32(want).view(np.uint32) & 0xFFFFE000).view(np.float32))
                if got != hi:
                    bad += 1
                    if bad < 5:
                        print(f"  B mismatch m {mm} c {cc}: got {got} want {want}")
    print("  B-tile mismatches:", bad)
    acc = d[16 + 65536:16 + 65536 + 128 * 256].view(np.float32).reshape(128, 256)
    ref = F.conv2d(x.double(), wt.double(), padding=pad).cpu().numpy()
    print("  acc[0,:4]", acc[0, :4], "acc[1,:4]", acc[1, :4])
    if f == 1 and L._tc.flattened:
        print("  ref[p0,m0..3]", ref[0, :4, 0, 0], "ref[p1]", ref[0, :4].reshape(4, -1)[:, 1])
        print("  y[p0,m0..3]", y[0, :4].reshape(4, -1)[:, 0].cpu().numpy())
    return True


if __name__ == "__main__":
    torch.cuda.set_device(0)
    run("1x1-tiny", 1, 16, 4, 8, 16, 1, 0, "tf32")
    run("1x1-tiny", 1, 16, 4, 8, 16, 1, 0, "tf32x3")
    run("3x3-a", 2, 32, 16, 16, 64, 3, 1, "tf32")
