# A/B of several builds (FRIR_LIB each of paper_2304_08052_b200/lib/libfrir_*.so, base first): stage times, config 5 (8192 rooms) and config 2
for c in "5 --rooms 8192" "2"; do
  for L in paper_2304_08052_b200/lib/libfrir_base.so paper_2304_08052_b200/lib/libfrir_v*.so; do
    FRIR_LIB=$L timeout 300 python tools/stage_time.py --cfg $c
  done
done
