#!/usr/bin/env bash
# One GPU measurement pass (run under gpurun from the repo root):
#   the GPU test suite, bench lines (config 2 default incl. e2e, the drop-in
#   call pattern and the CPU baselines; the reference arm; configs 3, 4, 5;
#   a 2-rank protocol run), the K1b ncu metric dump bench.py reads for
#   `roofline.traffic`, the config-2 launch list and an `ncu --set full`
#   capture of K1b.  Outputs land in gpurun_out/round/.
set -u
OUT=${OUT:-gpurun_out/round}
mkdir -p "$OUT"
export PATH=/usr/local/cuda/bin:$PATH
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > "$OUT/gpu.txt" 2>&1
timeout 2400 python -m pytest tests -m gpu -q > "$OUT/pytest_gpu.log" 2>&1; echo "pytest=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke=$?"
timeout 900 python bench.py > "$OUT/bench_config2.json" 2> "$OUT/bench_config2.err"; echo "bench=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > "$OUT/bench_reference.json" 2> "$OUT/bench_reference.err"; echo "ref=$?"
timeout 900 python bench.py --config 3 --steps 3 --warmup 1 > "$OUT/bench_config3.json" 2> "$OUT/bench_config3.err"; echo "c3=$?"
timeout 600 python bench.py --config 4 --steps 3 --warmup 1 > "$OUT/bench_config4.json" 2> "$OUT/bench_config4.err"; echo "c4=$?"
timeout 900 python bench.py --config 5 --steps 1 --warmup 1 > "$OUT/bench_config5.json" 2> "$OUT/bench_config5.err"; echo "c5=$?"
timeout 900 python bench.py --gpus 2 --same-device --steps 5 --warmup 2 --no-e2e --no-cpu > "$OUT/bench_2ranks_same_device.json" 2> "$OUT/bench_2ranks.err"; echo "mr=$?"
# K1b metric dump on the config-2 window (duration, DRAM bytes, warp instructions, issue)
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,lts__t_requests_srcunit_tex_op_red.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum \
  --clock-control none -k regex:scan_bpart -c 2 --csv --log-file "$OUT/ncu_metrics_bpart.csv" \
  python tools/sweep_k1p.py --reps 1 "" > /dev/null 2>&1; echo "ncu_metrics=$?"
# launch list of the default bench step (every kernel of the step)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k 'regex:sspd::|CUB_200802' -c 40 --csv \
  --log-file "$OUT/launches_config2.csv" python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
echo "launches=$?"
# full capture of the dominant kernel
timeout 900 ncu --set full --import-source on --clock-control none -k regex:scan_bpart -c 1 -f -o "$OUT/k1b_full" \
  python tools/sweep_k1p.py --reps 1 "" > /dev/null 2>&1; echo "ncu_full=$?"
# per-slide kernels of the sliding trace (slides ~50-75 of the warm-up step)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k 'regex:sspd::' -s 600 -c 300 --csv \
  --log-file "$OUT/launches_config4.csv" python bench.py --config 4 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1; echo "launches_c4=$?"

