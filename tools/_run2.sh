set -u
OUT=gpurun_out/r2a; mkdir -p $OUT
timeout 2400 python -m pytest tests/test_gpu_fullscale.py -x -q > $OUT/fullscale.log 2>&1; echo fullscale=$?; tail -3 $OUT/fullscale.log
timeout 600 python bench.py --steps 10 --warmup 3 > $OUT/bench2.json 2> $OUT/bench2.err; echo bench=$?
tail -c 3000 $OUT/bench2.json
