# A/B of the in-tree library against lib/libfrir_old.so (HEAD) on configs 5 (1024 rooms) and 2; then GPU tests
T=${1:-ab}
for c in "5 --rooms 1024" "2"; do
  for r in 1 2; do
  python tools/stage_time.py --cfg $c
  FRIR_LIB=paper_2304_08052_b200/lib/libfrir_old.so python tools/stage_time.py --cfg $c
  done
done 2>&1 | tee gpurun_out/${T}_stages.txt
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${T}_pytest.txt; tail -4 gpurun_out/${T}_pytest.txt
