# A/B against lib/libfrir_old.so (round-2 start) + sort-rank digests + GPU tests
T=${1:-ab}
python tools/render_digest.py > gpurun_out/${T}_d0.txt; FRIR_SORT_BALLOT=1 python tools/render_digest.py > gpurun_out/${T}_d1.txt
paste gpurun_out/${T}_d0.txt gpurun_out/${T}_d1.txt
for c in "5 --rooms 1024" "2"; do
  python tools/stage_time.py --cfg $c
  FRIR_LIB=paper_2304_08052_b200/lib/libfrir_old.so python tools/stage_time.py --cfg $c
done 2>&1 | tee gpurun_out/${T}_stages.txt
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${T}_pytest.txt; tail -2 gpurun_out/${T}_pytest.txt
