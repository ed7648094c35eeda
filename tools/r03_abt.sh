# quick GPU check of a kernel change: parity tests touching it, then tools/r03_ab.sh (A/B vs libfrir_base.so)
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_parity.py tests/test_gpu_parity_sweep.py 2>&1 | tail -3
bash tools/r03_ab.sh ${1:-ab}
