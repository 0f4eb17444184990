OUT=gpurun_out/c4b; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_sliding_dist.py -x -q -k "ring" > $OUT/pt.log 2>&1; echo pt=$?; tail -2 $OUT/pt.log
for v in 0 1; do
SSPD_SLIDE_PARTITIONED=$v timeout 600 python bench.py --config 4 --steps 3 --warmup 1 > $OUT/bench4_$v.json 2> $OUT/bench4_$v.err; echo c4_$v=$?
python -c "
import json; d=json.loads(open('$OUT/bench4_$v.json').read().strip().splitlines()[-1]); print($v, d['value'], d['ms_per_step'], d['step_ms'], d['detect'])"
done
SSPD_SLIDE_PARTITIONED=1 timeout 600 python tools/timeline_config4.py > $OUT/timeline.txt 2>&1; tail -12 $OUT/timeline.txt
