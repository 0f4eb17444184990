#!/usr/bin/env bash
# One GPU measurement pass (run under gpurun from the repo root):
#   bench lines (config 2 default incl. e2e + CPU baseline, reference arm,
#   config 4, config 5), the K1p ncu metric dump that bench.py reads for
#   `roofline.traffic`, the config-2 launch list and an `ncu --set full`
#   capture of K1p.  Outputs land in gpurun_out/round/.
set -u
OUT=gpurun_out/round
mkdir -p "$OUT"
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/gpu.txt" 2>&1
timeout 900 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest=$?"
timeout 600 python bench.py > "$OUT/bench_config2.json" 2> "$OUT/bench_config2.err"; echo "bench=$?"
timeout 600 python bench.py --impl reference > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"; echo "ref=$?"
timeout 900 python bench.py --config 3 --steps 3 --warmup 1 > "$OUT/bench_config3.json" 2> "$OUT/bench_config3.err"; echo "c3=$?"
timeout 600 python bench.py --config 4 --steps 3 --warmup 1 > "$OUT/bench_config4.json" 2> "$OUT/bench_config4.err"; echo "c4=$?"
# config-4 launch list inside the timed step (the warmup step is ~5,000 launches)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled --launch-skip 3600 -c 180 --csv \
  --log-file "$OUT/launches_config4.csv" python bench.py --config 4 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
echo "launches4=$?"
timeout 900 python bench.py --config 5 --steps 1 --warmup 1 > "$OUT/bench_config5.json" 2> "$OUT/bench_config5.err"; echo "c5=$?"
# K1p metric dump on the config-2 window (duration, DRAM bytes, warp instructions)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_requests_srcunit_tex_op_red.sum \
  --clock-control none -k regex:scan_partitioned -c 2 --csv --log-file "$OUT/ncu_metrics_partitioned.csv" \
  python tools/sweep_k1p.py --reps 1 "" > /dev/null 2>&1; echo "ncu_metrics=$?"
# launch list of the default bench step (every kernel of the step)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k 'regex:sspd::|CUB_200802' -c 66 --csv \
  --log-file "$OUT/launches_config2.csv" python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
echo "launches=$?"
# full capture of the dominant kernel
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_partitioned -c 1 -f -o "$OUT/k1p_full" \
  python tools/sweep_k1p.py --reps 1 "" > /dev/null 2>&1; echo "ncu_full=$?"
# full captures of the config-4 scan (deferred) and the restore (K5, warp per SEA)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_sliding_u16_fast --launch-skip 400 -c 1 -f \
  -o "$OUT/k2_deferred_full" python bench.py --config 4 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1; echo "ncu_k2=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:restore_warp --launch-skip 150 -c 1 -f \
  -o "$OUT/restore_full" python bench.py --config 4 --steps 1 --warmup 0 --no-cpu > /dev/null 2>&1; echo "ncu_restore=$?"
