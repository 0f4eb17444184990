OUT=gpurun_out/p10; mkdir -p $OUT
timeout 1200 python tools/sweep_k1p.py --reps 6 "" "SSPD_BPART_CONS_WARPS=4" "SSPD_BPART_CONS_WARPS=6" "SSPD_BPART_CONS_WARPS=4,SSPD_PART_WEIGHT=68" "SSPD_BPART_CONS_WARPS=6,SSPD_PART_WEIGHT=70" > $OUT/sweep.jsonl 2> $OUT/sweep.err
cat $OUT/sweep.jsonl; tail -3 $OUT/sweep.err
