# A/B of several builds over the given configs (default: 5 at 8192 rooms, 2, 3, 4): stage times per build
CFGS=${CFGS:-"5 --rooms 8192|2|3|4"}
IFS='|' read -ra CS <<< "$CFGS"
for c in "${CS[@]}"; do
  for L in paper_2304_08052_b200/lib/libfrir_base.so paper_2304_08052_b200/lib/libfrir_v*.so; do
    FRIR_LIB=$L timeout 300 python tools/stage_time.py --cfg $c
  done
done
