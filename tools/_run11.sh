OUT=gpurun_out/c4g; mkdir -p $OUT
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 python -m pytest tests/test_gpu_sliding_dist.py -x -q > $OUT/pt.log 2>&1; echo pt=$?; tail -2 $OUT/pt.log
timeout 600 python bench.py --config 4 --steps 3 --warmup 1 > $OUT/b.json 2> $OUT/b.err; echo c4=$?
python -c "
import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['step_ms'], d['detect']['reports_total'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled --launch-skip 600 -c 60 --csv --log-file $OUT/launches_early.csv python bench.py --config 4 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1; echo early=$?
grep -h "scan_bpart\|sliding" $OUT/launches_early.csv | head -4 | awk -F'","' '{print $5, $(NF-1), $NF}' | cut -c1-150
