T=${1:-ab}
for c in "5 --rooms 1024" "2" "3 --rooms 512"; do
  python tools/stage_time.py --cfg $c
  FRIR_SORT_NW=8 python tools/stage_time.py --cfg $c
  FRIR_SORT_NW=16 python tools/stage_time.py --cfg $c
done 2>&1 | tee gpurun_out/${T}_stages.txt
