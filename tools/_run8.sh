OUT=gpurun_out/p5; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "partitioned" > $OUT/pt.log 2>&1; echo pt=$?; tail -2 $OUT/pt.log
SSPD_BPART_CONS=2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "partitioned" > $OUT/pt2.log 2>&1; echo pt2=$?; tail -2 $OUT/pt2.log
timeout 900 python tools/sweep_k1p.py --reps 5 "" "SSPD_BPART_CONS=0" "SSPD_BPART_CONS=2" "SSPD_BPART_CONS=1,SSPD_BPART_TILES=32" > $OUT/sweep.jsonl 2> $OUT/sweep.err
cat $OUT/sweep.jsonl; tail -3 $OUT/sweep.err
