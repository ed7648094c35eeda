# config-5 launch size sweep (value, one stream) + GPU tests
for ch in 2048 4096 8192; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --chunk $ch > gpurun_out/ch_$ch.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ch_$ch.json')); print('chunk $ch', round(d['value']), d['stages']['serial_ms_per_step'], d['stages']['value_streams'])"
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
