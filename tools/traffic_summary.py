"""Summarise tools/gemm_traffic.sh captures into profiles/<round>/gemm_traffic.json:
per shape, DRAM read+write of the one measured launch against its algorithmic
bytes, the launch duration and DRAM throughput (cold L2, serialised: ncu)."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tools.gemm_traffic import SHAPES, algorithmic_bytes  # noqa: E402

METRICS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "dram__bytes_read.sum.pct_of_peak_sustained_elapsed", "launch__grid_size", "Kernel Name"]


def read(path):
    path = Path(path)
    if path.suffix == ".csv":
        out = path.read_text()
    else:
        out = subprocess.run(["ncu", "-i", str(path), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            d[m] = (vals[i], units[i])
    return d


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


def to_us(v, u):
    v = float(v.replace(",", ""))
    return v * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(u, 1)


def main(src, dst):
    res = {"source": "ncu --set full --clock-control none --nvtx --nvtx-include measure/ -k regex:gemm_streamk "
                     "python tools/gemm_traffic.py run <shape> (one launch after a 256 MB L2 flush)",
           "shapes": {}}
    for name, (n_tok, n_out, k) in SHAPES.items():
        rep = Path(src) / f"{name}.csv"
        if not rep.exists():
            rep = Path(src) / f"{name}.ncu-rep"
        if not rep.exists():
            continue
        d = read(rep)
        rd = to_bytes(*d["dram__bytes_read.sum"])
        wr = to_bytes(*d["dram__bytes_write.sum"])
        us = to_us(*d["gpu__time_duration.sum"])
        alg = algorithmic_bytes(n_tok, n_out, k)
        res["shapes"][name] = {"n_tok": n_tok, "n_out": n_out, "k": k, "kernel": d["Kernel Name"][0],
                               "dram_read": rd, "dram_write": wr, "algorithmic_bytes": alg,
                               "traffic_over_algorithmic": round((rd + wr) / alg, 4), "ncu_us": us,
                               "ncu_GBps_algorithmic": round(alg / us / 1e3, 1),
                               "dram_pct_peak": float(d["dram__bytes_read.sum.pct_of_peak_sustained_elapsed"][0])}
    s7 = [v for n, v in res["shapes"].items() if n.startswith("7b_") and "lm_head" not in n]
    if s7:
        res["traffic_bytes_per_launch_avg_7b_layer"] = sum(v["dram_read"] + v["dram_write"] for v in s7) / len(s7)
        res["algorithmic_bytes_per_launch_avg_7b_layer"] = sum(v["algorithmic_bytes"] for v in s7) / len(s7)
    Path(dst).write_text(json.dumps(res, indent=1) + "\n")
    for n, v in res["shapes"].items():
        print(f"{n:18s} traffic/alg {v['traffic_over_algorithmic']:.3f}  {v['ncu_us']:8.2f} us  "
              f"{v['ncu_GBps_algorithmic']:7.1f} GB/s  dram {v['dram_pct_peak']:.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
