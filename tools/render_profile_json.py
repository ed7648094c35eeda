"""Write profiles/render_ncu.json (read by bench.py's roofline) from an
`ncu --set full` report of one render launch -- the render_kernel launches of one batch (dev tool).

usage: python tools/render_profile_json.py REPORT.ncu-rep CFG ROOMS_PER_LAUNCH [SOURCE_NOTE]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

rep, cfg, rooms = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
note = sys.argv[4] if len(sys.argv) > 4 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
# one render launch = the full + early sweep, or (split batches) the full pass
# and the early pass: sum the render_kernel rows of the capture
recs = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if "render_kernel" in d.get("Kernel Name", ""):
        recs.append(d)
if not recs:
    sys.exit("no render_kernel in the report")


def val(d, k):
    return float(d[k].replace(",", "")) * scale.get(units[hdr.index(k)], 1.0)


def tot(k):
    return sum(val(d, k) for d in recs)


dur = tot("gpu__time_duration.sum")
out_path = Path(__file__).resolve().parents[1] / "profiles" / "render_ncu.json"
allp = json.loads(out_path.read_text()) if out_path.exists() else {}
allp[f"cfg{cfg}"] = {
    "rooms_per_launch": rooms,
    "kernels": [d["Kernel Name"] for d in recs],
    "dram_bytes": tot("dram__bytes_read.sum") + tot("dram__bytes_write.sum"),
    "duration_s": dur,
    # time-weighted over the kernels of the launch
    "fp32_pipe_pct": sum(val(d, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active") *
                         val(d, "gpu__time_duration.sum") for d in recs) / dur,
    "issue_active_pct": sum(val(d, "smsp__issue_active.avg.pct_of_peak_sustained_active") *
                            val(d, "gpu__time_duration.sum") for d in recs) / dur,
    "inst_executed": tot("smsp__inst_executed.sum"),
    "shared_wavefronts": tot("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "source": note,
}
out_path.write_text(json.dumps(allp, indent=1) + "\n")
print(json.dumps(allp[f"cfg{cfg}"], indent=1))
