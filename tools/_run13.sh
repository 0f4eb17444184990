OUT=gpurun_out/c4j; mkdir -p $OUT
export PATH=/usr/local/cuda/bin:$PATH
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py tests/test_gpu_sliding_dist.py -x -q -k "not config2_full" > $OUT/pt.log 2>&1; echo pt=$?; tail -2 $OUT/pt.log
timeout 600 python bench.py --config 4 --steps 3 --warmup 1 > $OUT/b.json 2> $OUT/b.err; echo c4=$?
python -c "
import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['step_ms'], d['detect']['reports_total'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:restore_warp --launch-skip 280 -c 3 --csv --log-file $OUT/restore.csv python bench.py --config 4 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1; echo r=$?
grep -h "duration" $OUT/restore.csv | awk -F'","' '{print $(NF-1), $NF}'
