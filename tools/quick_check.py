"""Quick GPU correctness probe (development aid): both engines vs the oracle."""
import sys, time, json
import numpy as np
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import oracle
import paper_2103_16234_b200 as pk

cases = [
    ("c1", 1, 64, 56, 56, 64, 3, 3, 1, 1, 1),
    ("t1", 1, 1, 1, 1, 1, 1, 1, 1, 0, 0),
    ("t2", 2, 3, 5, 7, 5, 3, 3, 1, 1, 1),
    ("t3", 2, 20, 7, 7, 33, 1, 1, 1, 0, 0),
    ("5x5", 3, 17, 7, 7, 40, 5, 5, 1, 2, 2),
    ("s2", 2, 9, 13, 11, 20, 3, 3, 2, 1, 1),
    ("7x7s2", 1, 3, 40, 40, 64, 7, 7, 2, 3, 3),
    ("even", 2, 5, 9, 8, 7, 2, 4, 1, 1, 2),
    ("1x1s2", 2, 30, 14, 14, 70, 1, 1, 2, 0, 0),
    ("g1x1", 4, 192, 28, 28, 16, 1, 1, 1, 0, 0),
]
ok = True
for name, n, c, h, w, m, hf, wf, s, ph, pw in cases:
    cfg = pk.ConvConfig(name, n=n, c=c, h=h, w=w, m=m, hf=hf, wf=wf, stride=s, pad_h=ph, pad_w=pw)
    x = pk.make_tensor(pk.input_dims(cfg), "uniform", seed=11)
    f = pk.make_tensor(pk.filter_dims(cfg), "uniform", seed=12)
    ref64 = oracle.conv_f64(cfg, x.data, f.data)
    naive = oracle.conv_naive(cfg, x.data, f.data)
    out = pk.conv_forward(x, f, cfg).data
    err = oracle.relative_error(out, ref64)
    tol = oracle.fp32_tolerance(c, hf, wf)
    line = {"case": name, "fused_err": err, "tol": tol, "fused_ok": err <= tol,
            "tiles": pk.select_tiles(cfg).family}
    if s == 1:
        o2, st = pk.conv_twostage(x, f, cfg)
        line["twostage_bitwise"] = o2.data.tobytes() == naive.tobytes()
        line["twostage_err"] = oracle.relative_error(o2.data, ref64)
        ok &= line["twostage_bitwise"]
    ok &= line["fused_ok"]
    print(json.dumps(line), flush=True)
print("ALL_OK" if ok else "FAILURES")
