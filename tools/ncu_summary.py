"""Readable summary of an ncu report (--set full): key raw metrics + the
details page (section | metric | unit | value), for committing under profiles/.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/rNN/<name>.txt
"""
import csv
import io
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tensor.sum", "launch__grid_size", "launch__block_size",
       "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "lts__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def run(page, path):
    out = subprocess.run(["ncu", "-i", path, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(path):
    raw = run("raw", path)
    if len(raw) >= 3:
        hdr, units = raw[0], raw[1]
        for row in raw[2:]:
            name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
            print(f"== kernel: {name}")
            for m in RAW:
                for i, h in enumerate(hdr):
                    if h == m:
                        print(f"  {m:65s} {row[i]:>16s} {units[i]}")
    det = run("details", path)
    if det:
        hdr = det[0]
        ix = {k: hdr.index(k) for k in ("Section Name", "Metric Name", "Metric Unit", "Metric Value") if k in hdr}
        print("\n== details")
        for row in det[1:]:
            if len(row) > max(ix.values()) and row[ix["Metric Name"]]:
                print(f"  {row[ix['Section Name']][:34]:34s} | {row[ix['Metric Name']][:48]:48s} | "
                      f"{row[ix['Metric Unit']]:10s} | {row[ix['Metric Value']]}")


if __name__ == "__main__":
    main(sys.argv[1])
