set -x
mkdir -p gpurun_out/v8
python bench.py > gpurun_out/v8/bench_cfg2.json 2> gpurun_out/v8/bench_cfg2.err
for c in 1 3 4 5; do timeout 900 python bench.py --config $c > gpurun_out/v8/bench_cfg$c.json 2> gpurun_out/v8/bench_cfg$c.err; done
timeout 900 python bench.py --impl reference > gpurun_out/v8/bench_reference_arm.json 2> gpurun_out/v8/ref.err
timeout 900 python bench_rows.py > gpurun_out/v8/bench_rows.json 2> gpurun_out/v8/rows.err
timeout 900 python bench_mix.py > gpurun_out/v8/bench_mix.json 2> gpurun_out/v8/mix.err
ncu --set full --clock-control none --import-source on -k regex:"geom_kernel|sort_kernel|tail_kernel|render_kernel" -c 4 -f -o gpurun_out/v8/cfg2 python tools/prof_cfg.py --cfg 2 --iters 1 > gpurun_out/v8/ncu_cfg2.log 2>&1
ncu --set full --clock-control none -k regex:"geom_kernel|sort_kernel|tail_kernel|render_kernel|seam_kernel" -c 6 -f -o gpurun_out/v8/ism python tools/stage_time.py --ism 128 --reps 1 > gpurun_out/v8/ncu_ism.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/v8/bench_cfg2_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/v8/rows_launches.csv python bench_rows.py --no-cpu-baseline --steps 2 --warmup 1 > /dev/null 2>&1
ls -la gpurun_out/v8
