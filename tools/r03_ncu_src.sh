# ncu --set full with source-level SASS counters for each kernel of a 1024-room config-5 launch
T=${1:-src}
timeout 1200 ncu --set full --import-source on --clock-control none -k "regex:geom_kernel|sort_kernel|tail_kernel|render_kernel" -c 4 \
  -o gpurun_out/${T}_cfg5 python tools/prof_cfg.py --cfg 5 --rooms 1024 --iters 0 > gpurun_out/${T}_ncu.log 2>&1
tail -3 gpurun_out/${T}_ncu.log
