"""Summarise an ncu DRAM-traffic capture of the bench's lambda path into profiles/ncu_traffic.json.

    python tools/traffic_summary.py gpurun_out/traffic.csv gpurun_out/ncu_fits.json profiles/ncu_traffic.json
"""
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import algorithmic_bytes  # noqa: E402

csv_path, fits_path, out_path = sys.argv[1:4]
rows = {}
kernels = set()
with open(csv_path) as f:
    lines = [ln for ln in f if not ln.startswith("==")]
for r in csv.DictReader(lines):
    rows.setdefault(int(r["ID"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    kernels.add(r["Kernel Name"].split("(")[0].replace("void ", ""))
fits = json.load(open(fits_path))
p = fits["p"]
per = []
for i, fit in enumerate(fits["fits"]):
    m = rows[i]
    traffic = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    alg = algorithmic_bytes(p, fit["nnz_per_sweep"])
    per.append({"lam": fit["lam"], "iterations": fit["iterations"], "dram_bytes": traffic, "algorithmic_bytes": alg,
                "traffic_over_algorithmic": traffic / alg, "ncu_ms": m["gpu__time_duration.sum"] / 1e6})
    print(f"lam={fit['lam']:.2f} iters={fit['iterations']:3d} dram={traffic / 1e9:8.2f} GB "
          f"alg={alg / 1e9:8.2f} GB ratio={traffic / alg:5.2f} ncu={m['gpu__time_duration.sum'] / 1e6:8.1f} ms")
avg_traffic = sum(x["dram_bytes"] for x in per) / len(per)
avg_alg = sum(x["algorithmic_bytes"] for x in per) / len(per)
workload = f"ar2 p={p} n={fits['n']} lambda-path cold"
out = {workload: {"dram_bytes_per_launch": avg_traffic, "algorithmic_bytes_per_launch": avg_alg,
                  "kernel": ", ".join(sorted(kernels)), "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                  "(one launch per lambda of the bench path, kernel replay)", "per_fit": per}}
json.dump(out, open(out_path, "w"), indent=1)
print(f"average per launch: dram {avg_traffic / 1e9:.2f} GB, algorithmic {avg_alg / 1e9:.2f} GB")
