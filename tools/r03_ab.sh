# A/B of two builds: stage times (config 5, 8192 rooms incl. an I = 8192 room; config 2) + headline bench of the new build
for c in "5 --rooms 8192" "2"; do
  for L in paper_2304_08052_b200/lib/libfrir_base.so paper_2304_08052_b200/lib/libfrir.so; do
    FRIR_LIB=$L timeout 300 python tools/stage_time.py --cfg $c
  done
done
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${1:-ab}_cfg5.json 2> gpurun_out/${1:-ab}_cfg5.err
python -c "import json; d=json.load(open('gpurun_out/${1:-ab}_cfg5.json')); print('cfg5', d['value'], d['stages'])"
