OUT=gpurun_out/p14; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "partitioned" > $OUT/pt.log 2>&1; echo pt=$?; tail -2 $OUT/pt.log
timeout 900 python tools/sweep_k1p.py --reps 6 "" "SSPD_BPART_DRAIN_DEPTH=0" "SSPD_BPART_DRAIN_DEPTH=4" "SSPD_BPART_DRAIN_DEPTH=8" "SSPD_BPART_CONS_WARPS=6" "SSPD_BPART_CONS_WARPS=6,SSPD_PART_WEIGHT=68" "SSPD_BPART_CONS_WARPS=4,SSPD_PART_WEIGHT=66" "SSPD_BPART_CONS=3" > $OUT/sweep.jsonl 2> $OUT/sweep.err
cat $OUT/sweep.jsonl; tail -3 $OUT/sweep.err
