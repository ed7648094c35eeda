# full GPU suite (incl. the parity sweep, record -> gpurun_out/parity_r02.json) + the headline bench line
T=${1:-t}
nproc
FRIR_PARITY_OUT=gpurun_out/parity_r02.json timeout 2400 python -m pytest tests -m gpu -q -x --durations=8 > gpurun_out/${T}_pytest.txt 2>&1; tail -15 gpurun_out/${T}_pytest.txt
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_cfg5.json 2> gpurun_out/${T}_cfg5.err
python -c "import json; d=json.load(open('gpurun_out/${T}_cfg5.json')); print('cfg5', d['value'], d['stages'])" || tail -20 gpurun_out/${T}_cfg5.err
