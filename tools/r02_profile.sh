# ncu evidence for the headline (config 5): launch list of the bench command and
# one --set full capture of each kernel of a 4096-room launch (the bench's launch size)
T=${1:-prof}
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_bench.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:geom_kernel|sort_kernel|tail_kernel|render_kernel" -c 4 \
  -o gpurun_out/${T}_cfg5 python tools/prof_cfg.py --cfg 5 --rooms 4096 --iters 0 > gpurun_out/${T}_ncu_full.log 2>&1
tail -2 gpurun_out/${T}_ncu_full.log; ls -la gpurun_out | grep $T
