OUT=gpurun_out/c4; mkdir -p $OUT
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python bench.py --config 4 --steps 3 --warmup 1 > $OUT/bench4.json 2> $OUT/bench4.err; echo c4=$?
python -c "
import json; d=json.loads(open('$OUT/bench4.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['step_ms'], d['scan_roofline'])"
timeout 600 python tools/timeline_config4.py > $OUT/timeline.txt 2>&1; tail -24 $OUT/timeline.txt
timeout 300 python tools/host_overhead_config4.py > $OUT/host.txt 2>&1; cat $OUT/host.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled --launch-skip 3600 -c 180 --csv --log-file $OUT/launches_config4.csv python bench.py --config 4 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1; echo launches=$?
