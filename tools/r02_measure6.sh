# Round-2 measurement set (m6: final build, 2-deep pipeline, early pass from 1,024 channels): headline bench (config 5) + reference arm, configs 1-4, ncu launch list and
# one --set full capture of each kernel of a 4096-room config-5 launch.  Outputs: gpurun_out/${T}_*
T=${1:-m}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv,noheader
timeout 900 python bench.py > gpurun_out/${T}_cfg5.json 2> gpurun_out/${T}_cfg5.err
timeout 900 python bench.py --impl reference > gpurun_out/${T}_ref_cfg5.json 2> gpurun_out/${T}_ref_cfg5.err
for c in 1 2 3 4; do timeout 900 python bench.py --config $c > gpurun_out/${T}_cfg$c.json 2> gpurun_out/${T}_cfg$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:geom_kernel|sort_kernel|tail_kernel|render_kernel" -c 5 \
  -o gpurun_out/${T}_cfg5_full python tools/prof_cfg.py --cfg 5 --rooms 4096 --iters 0 > gpurun_out/${T}_ncu_full.log 2>&1
python - "$T" << 'PY'
import json, sys
t = sys.argv[1]
for c in ("cfg5", "ref_cfg5", "cfg1", "cfg2", "cfg3", "cfg4"):
    try:
        d = json.loads(open(f"gpurun_out/{t}_{c}.json").read().strip().splitlines()[-1])
        print(c, "value %.1f" % d["value"], "e2e %.1f" % d["e2e"]["value"], "cpu", (d.get("cpu_baseline") or {}).get("value"),
              "frac", (d.get("roofline") or {}).get("frac"), "clocks", d.get("clocks"))
    except Exception as e:
        print(c, "FAILED", e)
PY
