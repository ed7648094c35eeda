# render residency experiment: pipelined bench value with 3 (default) vs 2 render CTAs per SM
T=${1:-ab}
for v in 0 2; do
  FRIR_RENDER_CTAS=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ctas$v.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/${T}_ctas$v.json')); print('ctas=$v', round(d['value']), d['stages']['serial_ms_per_step'], d['stages']['render_ms_per_step'])"
done
