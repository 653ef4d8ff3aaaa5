"""Measured DRAM traffic per layer for bench.py's roofline (GPU box, under ncu).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none -k regex:"conv|stage2|pack" --csv --log-file gpurun_out/tr/ncu.csv \
        python tools/traffic.py run c1,c2,c3,c4,c5 > gpurun_out/tr/layers.json
    python tools/traffic.py merge gpurun_out/tr/layers.json gpurun_out/tr/ncu.csv > profiles/r1_traffic.json

`run` launches every layer of each workload once, at bench.py's default batch
and with the plan bench.py uses (fused engine), and prints the ordered list of
(workload, layer, plan, expected b2c launches).  `merge` walks ncu's launch
list in the same order and sums the DRAM bytes of each layer's launches (conv
kernel + split-C stage-2 sum + the packed path's pixel gather): the "traffic" bench.py reports next to the
algorithmic bytes.  ncu replays each kernel with caches flushed, so these are
cold-cache bytes per launch.
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(workloads):
    import torch

    import bench
    from paper_2103_16234_b200 import ConvLayer
    from paper_2103_16234_b200 import workloads as W

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    order = []
    for wl in workloads:
        cfgs = W.layers(wl, bench.DEFAULT_BATCH[wl])
        xs, ws, ys = bench.make_operands(cfgs, dev, 0)
        torch.cuda.synchronize()
        for c, x, w, y in zip(cfgs, xs, ws, ys):
            L = ConvLayer(c, "fused")
            L(x, w, out=y)
            torch.cuda.synchronize()
            n = (2 if (L.splits > 1 and L.reduce != 2) else 1) + (1 if "1x1pk" in L.family else 0)  # + pixel packing
            order.append({"workload": wl, "layer": c.name, "family": L.family, "launches": n,
                          "alg_bytes": c.compulsory_bytes, "flops": c.flops})
        del xs, ws, ys
        torch.cuda.empty_cache()
    print(json.dumps(order))


def merge(layers_path, ncu_csv):
    order = json.loads([l for l in open(layers_path) if l.startswith("[")][-1])
    with open(ncu_csv) as fh:
        lines = [l for l in fh if not l.startswith("==")]
    per = {}
    for r in csv.DictReader(io.StringIO("".join(lines))):
        k = int(r["ID"])
        e = per.setdefault(k, {"name": r["Kernel Name"], "bytes": 0.0, "us": 0.0})
        v = float(r["Metric Value"].replace(",", "") or 0)
        unit = r.get("Metric Unit", "")
        if r["Metric Name"].startswith("dram__bytes"):
            e["bytes"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif r["Metric Name"] == "gpu__time_duration.sum":
            e["us"] += v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(unit, 1)
    launches = [per[k] for k in sorted(per)]
    need = sum(o["launches"] for o in order)
    if len(launches) != need:
        raise SystemExit(f"ncu saw {len(launches)} b2c launches, the layer list expects {need}")
    out, i = {}, 0
    for o in order:
        ks = launches[i:i + o["launches"]]
        i += o["launches"]
        out.setdefault(o["workload"], {})[o["layer"]] = {
            "family": o["family"], "dram_bytes": round(sum(k["bytes"] for k in ks)),
            "alg_bytes": o["alg_bytes"], "us_cold": round(sum(k["us"] for k in ks), 2),
            "kernels": [k["name"].split("(")[0] for k in ks]}
    out["_source"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                      "--clock-control none (cache flushed per replay); tools/traffic.py")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2].split(","))
    else:
        merge(sys.argv[2], sys.argv[3])
