T=${1:-st}
timeout 900 python -m pytest tests/test_gpu_stages.py -q -x 2>&1 | tail -30 > gpurun_out/${T}_stages.txt; tail -30 gpurun_out/${T}_stages.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -8 > gpurun_out/${T}_pytest.txt; tail -4 gpurun_out/${T}_pytest.txt
