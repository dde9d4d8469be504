"""One line per kernel of an ncu --set full report: duration, DRAM bytes, tensor /
SM / memory throughput, L2 hit rate, achieved occupancy, top stall reasons."""
import csv
import io
import subprocess
import sys

if sys.argv[1].endswith((".csv", ".csv.gz")):  # raw page exported on the GPU box (ncu -i X --page raw --csv)
    import gzip

    raw = (gzip.open if sys.argv[1].endswith(".gz") else open)(sys.argv[1], "rt").read()
else:
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def g(r, name):
    i = col.get(name)
    if i is None or not r[i]:
        return None
    try:
        return float(r[i].replace(",", ""))
    except ValueError:
        return r[i]


stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
print("| kernel | grid | us | DRAM MB | tensor % | SM % | mem % | L2 hit % | occ % | top stalls (per issue) |")
print("|---|---|---|---|---|---|---|---|---|---|")
for r in data:
    name = r[col["Kernel Name"]].split("(")[0].replace("smpm::", "")
    dur = g(r, "gpu__time_duration.sum")
    dram = (g(r, "dram__bytes_read.sum") or 0) + (g(r, "dram__bytes_write.sum") or 0)
    du = units[col["dram__bytes_read.sum"]]
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(du, 1.0)
    st = sorted(((g(r, h) or 0.0, h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                 for h in stalls), reverse=True)
    st = ", ".join(f"{n} {v:.1f}" for v, n in st if n != "selected")[:90]
    tens = g(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")
    print(f"| {name} | {r[col['Grid Size']]} | {dur:.1f} | {dram * scale:.1f} | {tens if tens is not None else 0:.1f} | "
          f"{g(r, 'sm__throughput.avg.pct_of_peak_sustained_elapsed') or 0:.1f} | "
          f"{g(r, 'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed') or 0:.1f} | "
          f"{g(r, 'lts__t_sector_hit_rate.pct') or 0:.1f} | "
          f"{g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active') or 0:.1f} | {st} |")
