# value schedules: one stream, 2-stream pipeline, split (pre-render high priority / render low priority)
for c in 5 2; do
  for s in 1 2 split; do
    FRIR_BENCH_SCHED=$s timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sched_${c}_$s.json 2> gpurun_out/sched_${c}_$s.err
    python -c "import json; d=json.load(open('gpurun_out/sched_${c}_$s.json')); print('cfg $c sched $s', round(d['value']), round(d['ms_per_step'], 3))" || tail -3 gpurun_out/sched_${c}_$s.err
  done
done
