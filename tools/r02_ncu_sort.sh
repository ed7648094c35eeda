# ncu --set full of the sort + tail kernels of one config-5 launch (1024 rooms)
T=${1:-sortprof}
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:sort_kernel|tail_kernel" -c 2 \
  -o gpurun_out/${T}_cfg5 python tools/prof_cfg.py --cfg 5 --rooms 1024 --iters 0 > gpurun_out/${T}_ncu.log 2>&1
tail -2 gpurun_out/${T}_ncu.log
