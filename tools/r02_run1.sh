set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r1_pytest.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench_cfg5.json 2> gpurun_out/r1_bench_cfg5.err
timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_cfg2.json 2> gpurun_out/r1_bench_cfg2.err
timeout 600 python bench.py --gpus 2 --dist-backend gloo --rooms 16384 --steps 3 --warmup 3 > gpurun_out/r1_bench_2rank.json 2> gpurun_out/r1_bench_2rank.err
tail -3 gpurun_out/*.err
cat gpurun_out/r1_pytest.txt
