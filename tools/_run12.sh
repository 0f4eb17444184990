OUT=gpurun_out/p15; mkdir -p $OUT
timeout 900 python tools/sweep_k1p.py --reps 6 "" "SSPD_BPART_PREFETCH=1" "SSPD_BPART_PREFETCH=1,SSPD_BPART_TILES=24" "SSPD_BPART_PREFETCH=1,SSPD_BPART_CONS_WARPS=6" > $OUT/sweep.jsonl 2> $OUT/sweep.err
cat $OUT/sweep.jsonl; tail -3 $OUT/sweep.err
