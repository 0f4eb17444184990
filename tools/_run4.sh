set -u
OUT=gpurun_out/r2c; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_multiproc.py tests/test_gpu_refshim.py -x -q > $OUT/pt.log 2>&1; echo pt=$?; tail -3 $OUT/pt.log
timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu > $OUT/bench2.json 2> $OUT/bench2.err; echo bench=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/r2c/bench2.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e'].get('dropin'))
PY
