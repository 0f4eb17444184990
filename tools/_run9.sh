OUT=gpurun_out/p6; mkdir -p $OUT
export PATH=/usr/local/cuda/bin:$PATH
SSPD_BPART_FLUSH_TMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "partitioned" > $OUT/pt.log 2>&1; echo pt=$?; tail -2 $OUT/pt.log
timeout 900 python tools/sweep_k1p.py --reps 5 "" "SSPD_BPART_FLUSH_TMA=1" "SSPD_BPART_TILES=8" "SSPD_BPART_TILES=8,SSPD_BPART_FLUSH_TMA=1" "SSPD_BPART_TILES=4" "SSPD_BPART_TILES=4,SSPD_BPART_FLUSH_TMA=1" > $OUT/sweep.jsonl 2> $OUT/sweep.err
cat $OUT/sweep.jsonl; tail -3 $OUT/sweep.err
for t in 8 16; do
SSPD_BPART_TILES=$t timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:scan_bpart -c 1 --csv --log-file $OUT/ncu_t$t.csv python tools/sweep_k1p.py --reps 1 "" > /dev/null 2>&1; echo ncu$t=$?
grep -h "dram__bytes\|duration" $OUT/ncu_t$t.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
