set -u
OUT=gpurun_out/p2; mkdir -p $OUT
export PATH=/usr/local/cuda/bin:$PATH
python -m pytest tests/test_gpu_parity.py -x -q -k "partitioned or config2" > $OUT/pt.log 2>&1; tail -2 $OUT/pt.log
python tools/sweep_k1p.py --reps 5 "" "SSPD_BPART_TILES=6" "SSPD_BPART_TILES=8" "SSPD_BPART_TILES=12" "SSPD_BPART_TILES=16" "SSPD_PART_WEIGHT=72" "SSPD_PART_WEIGHT=88" > $OUT/sweep.jsonl 2> $OUT/sweep.err
cat $OUT/sweep.jsonl
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_bpart -c 1 -f -o $OUT/k1b_full python tools/sweep_k1p.py --reps 1 "" > /dev/null 2>&1; echo ncu_full=$?
