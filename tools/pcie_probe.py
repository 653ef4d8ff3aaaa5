"""Host<->device copy bandwidth of this box (pinned buffers): H2D alone, D2H
alone and both directions at once on two streams -- the ceiling of bench.py's
e2e leg.   python tools/pcie_probe.py [GB]"""
import json, sys
import torch

gb = float(sys.argv[1]) if len(sys.argv) > 1 else 2.0
n = int(gb * 2**30 / 4)
h1 = torch.empty(n, dtype=torch.float32, pin_memory=True)
h2 = torch.empty(n, dtype=torch.float32, pin_memory=True)
d1 = torch.empty(n, device="cuda")
d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def both():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


bytes_ = n * 4
t_h2d = timed(lambda: d1.copy_(h1, non_blocking=True))
t_d2h = timed(lambda: h2.copy_(d2, non_blocking=True))
t_both = timed(both)
print(json.dumps({"bytes": bytes_, "h2d_gbs": round(bytes_ / t_h2d / 1e6, 1), "d2h_gbs": round(bytes_ / t_d2h / 1e6, 1),
                  "bidirectional_total_gbs": round(2 * bytes_ / t_both / 1e6, 1)}))
