# A/B timing vs lib/libfrir_old.so + the parity sweep record of the in-tree library
T=${1:-ab}
for c in "5 --rooms 1024" "2"; do
  for L in paper_2304_08052_b200/lib/libfrir.so paper_2304_08052_b200/lib/libfrir_old.so; do
    FRIR_LIB=$L python tools/stage_time.py --cfg $c
  done
done 2>&1 | tee gpurun_out/${T}_stages.txt
FRIR_PARITY_OUT=gpurun_out/${T}_parity.json timeout 1200 python -m pytest tests/test_gpu_parity_sweep.py tests/test_gpu_parity.py -q -x 2>&1 | tail -3
python -c "
import json; d=json.load(open('gpurun_out/${T}_parity.json'))
print({k: (v['max_err_full'], v['max_err_early'], v['direct_mismatches']) for k, v in d.items()})"
