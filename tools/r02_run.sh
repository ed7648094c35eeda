# usage: bash tools/r02_run.sh TAG  -> gpu tests + cfg5/cfg2 bench lines under gpurun_out/TAG_*
T=${1:-run}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.txt 2>&1; tail -3 gpurun_out/${T}_pytest.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_cfg5.json 2> gpurun_out/${T}_cfg5.err
timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_cfg2.json 2> gpurun_out/${T}_cfg2.err
python - "$T" << 'PY'
import json, sys
t = sys.argv[1]
for c in ("cfg5", "cfg2"):
    try:
        d = json.loads(open(f"gpurun_out/{t}_{c}.json").read())
        print(c, "value %.0f" % d["value"], "stages", {k: round(v, 3) for k, v in d["stages"].items() if k != "note"},
              "frac %.3f" % d["roofline"]["frac"], "e2e %.0f" % d["e2e"]["value"])
    except Exception as e:
        print(c, "FAILED", e); print(open(f"gpurun_out/{t}_{c}.err").read()[-2000:])
PY
