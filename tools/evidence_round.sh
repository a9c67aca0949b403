#!/bin/bash
# One call that produces a round's evidence on the GPU box (outputs under gpurun_out/<tag>_*):
# GPU test suite, bench lines (Wan2.2 with the input sweep and the CPU sample, Hunyuan, the reference arm,
# step time by head count), ncu launch list + full captures, compute-sanitizer logs.
TAG=${1:-r02}
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputests.log 2>&1; tail -2 gpurun_out/${TAG}_gputests.log
python bench.py > gpurun_out/${TAG}_bench_wan22.json 2> gpurun_out/${TAG}_bench_wan22.err; tail -c 400 gpurun_out/${TAG}_bench_wan22.json
python bench.py --workload hunyuan-720p > gpurun_out/${TAG}_bench_hunyuan.json 2> gpurun_out/${TAG}_bench_hunyuan.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_bench_reference.err
: > gpurun_out/${TAG}_step_by_heads.jsonl
for h in 40 20 10 5; do
  python bench.py --no-sweep --no-dense --no-cpu-baseline --heads $h 2>/dev/null | tail -1 >> gpurun_out/${TAG}_step_by_heads.jsonl
done
bash tools/profile_round.sh $TAG > gpurun_out/${TAG}_profile_round.log 2>&1
bash tools/sanitize_round.sh $TAG > /dev/null 2>&1
tail -5 gpurun_out/${TAG}_sanitizer.txt
