# ncu --set full of one render launch (config 5, 1024 rooms) with source-level SASS metrics
T=${1:-nr}
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:render_kernel" -c 1 -o gpurun_out/${T}_render python tools/prof_cfg.py --cfg 5 --rooms 1024 --iters 0 > gpurun_out/${T}_ncu.log 2>&1
tail -3 gpurun_out/${T}_ncu.log
