# A/B: in-tree library vs lib/libfrir_old.so (HEAD) and lib/libfrir_g6.so; digests must match
T=${1:-ab}
for L in paper_2304_08052_b200/lib/libfrir.so paper_2304_08052_b200/lib/libfrir_old.so paper_2304_08052_b200/lib/libfrir_g6.so; do
  FRIR_LIB=$L python tools/render_digest.py | tr '\n' ' '; echo
done
for c in "5 --rooms 1024" "2"; do
  for L in paper_2304_08052_b200/lib/libfrir.so paper_2304_08052_b200/lib/libfrir_old.so paper_2304_08052_b200/lib/libfrir_g6.so; do
    FRIR_LIB=$L python tools/stage_time.py --cfg $c
  done
done 2>&1 | tee gpurun_out/${T}_stages.txt
