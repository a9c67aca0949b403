#!/bin/bash
# ncu evidence for a round (run on the GPU box through gpurun, from the repo root):
#   1. launch list of the bench command (every kernel of `bench.py --steps 1 --warmup 3`, eager launches)
#   2. one `--set full` capture of each main kernel on 8 Wan2.2 heads (tools/one_layer.py) and of the
#      DiT prologue kernels (tools/dit_block_time.py)
# Outputs land in gpurun_out/<tag>_*; summarise them here with tools/ncu_summary.py and
# tools/ncu_full_summary.py (which also writes profiles/attention_traffic.json) and commit the
# summaries under profiles/.
set -u
TAG=${1:-r02}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-graph --no-dense --no-sweep --no-cpu-baseline > gpurun_out/${TAG}_bench_under_ncu.log 2>&1
for k in attend_tc_kernel error_table_tc_kernel route_kernel key_stats_kernel gram_tc_kernel seed_gram_kernel \
         assign_tc_kernel lloyd_step_kernel; do
  # -s: skip the launches of the warm-up call where a kernel launches many times per call
  SKIP=0
  case $k in assign_tc_kernel|lloyd_step_kernel) SKIP=2;; esac
  ncu --set full --clock-control none --import-source on -k regex:$k -s $SKIP -c 2 -f -o gpurun_out/${TAG}_$k \
      python tools/one_layer.py --heads 8 --calls 1 > gpurun_out/${TAG}_ncu_$k.log 2>&1
done
for k in qkv_prologue_kernel heads_to_tokens_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$k -c 1 -f -o gpurun_out/${TAG}_$k \
      python tools/dit_block_time.py --reps 1 > gpurun_out/${TAG}_ncu_$k.log 2>&1
done
ls -la gpurun_out/${TAG}_*
