OUT=gpurun_out/c4d; mkdir -p $OUT
for env in "SSPD_DETECT_SAME_STREAM=0" "SSPD_DETECT_SAME_STREAM=1" "SSPD_DETECT_SAME_STREAM=1 SSPD_SLIDE_PARTITIONED=0" "SSPD_DETECT_SAME_STREAM=0 SSPD_SLIDE_PARTITIONED=0"; do
env $env timeout 600 python bench.py --config 4 --steps 3 --warmup 1 > $OUT/b.json 2> $OUT/b.err; echo "$env rc=$?"
python -c "
import json; d=json.loads(open('$OUT/b.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['step_ms'], d['detect']['reports_total'])"
done
