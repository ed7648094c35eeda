for c in "5 --rooms 1024" "2"; do
  for L in paper_2304_08052_b200/lib/libfrir.so paper_2304_08052_b200/lib/libfrir_g5.so paper_2304_08052_b200/lib/libfrir_g4.so; do
    FRIR_LIB=$L python tools/stage_time.py --cfg $c
  done
done
