set -u
OUT=gpurun_out/r2b; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_dropin.py tests/test_gpu_multiproc.py -x -q > $OUT/pt.log 2>&1; echo pt=$?; tail -3 $OUT/pt.log
timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu > $OUT/bench2.json 2> $OUT/bench2.err; echo bench=$?
for c in 2 3 4 5; do
  timeout 600 python bench.py --config $c --gpus 2 --same-device --steps 2 --warmup 1 --no-e2e --no-cpu --packets 16777216 > $OUT/mr_c$c.json 2> $OUT/mr_c$c.err; echo mr$c=$?; tail -c 400 $OUT/mr_c$c.json; echo
done
