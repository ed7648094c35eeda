# A/B of pre-render variants on config 5 (1024 rooms) and config 2; then the GPU tests
T=${1:-ab}
for c in "5 --rooms 1024" "2"; do
  python tools/stage_time.py --cfg $c
  FRIR_MATCH=1 python tools/stage_time.py --cfg $c
  FRIR_NO_BIN=1 python tools/stage_time.py --cfg $c
  FRIR_NO_BIN=1 FRIR_MATCH=1 python tools/stage_time.py --cfg $c
done 2>&1 | tee gpurun_out/${T}_stages.txt
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${T}_pytest.txt; tail -4 gpurun_out/${T}_pytest.txt
