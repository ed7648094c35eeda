# A/B: in-tree library vs lib/libfrir_old.so (HEAD): digests and stage times, then GPU tests
T=${1:-ab}
for L in paper_2304_08052_b200/lib/libfrir.so paper_2304_08052_b200/lib/libfrir_old.so; do
  FRIR_LIB=$L python tools/render_digest.py | tr '\n' ' '; echo
done
for c in "5 --rooms 1024" "2" "4 --rooms 64"; do
  for L in paper_2304_08052_b200/lib/libfrir.so paper_2304_08052_b200/lib/libfrir_old.so; do
    FRIR_LIB=$L python tools/stage_time.py --cfg $c
  done
done 2>&1 | tee gpurun_out/${T}_stages.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${T}_pytest.txt; tail -2 gpurun_out/${T}_pytest.txt
