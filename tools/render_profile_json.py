"""Write profiles/render_ncu.json (read by bench.py's roofline) from an
`ncu --set full` report of one render launch (dev tool).

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
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if "render_kernel" not in d.get("Kernel Name", ""):
        continue
    def val(k):
        return float(d[k].replace(",", "")) * scale.get(units[hdr.index(k)], 1.0)
    out_path = Path(__file__).resolve().parents[1] / "profiles" / "render_ncu.json"
    allp = json.loads(out_path.read_text()) if out_path.exists() else {}
    allp[f"cfg{cfg}"] = {
        "rooms_per_launch": rooms,
        "dram_bytes": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
        "duration_s": val("gpu__time_duration.sum"),
        "fp32_pipe_pct": val("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": val("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "inst_executed": val("smsp__inst_executed.sum"),
        "shared_wavefronts": val("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "source": f"{note}: ncu --set full --clock-control none, one render launch",
    }
    out_path.write_text(json.dumps(allp, indent=1) + "\n")
    print(json.dumps(allp[f"cfg{cfg}"], indent=1))
    break
