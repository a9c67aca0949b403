timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
run() { python bench.py --no-sweep --no-cpu-baseline --steps 5 --warmup 3 $2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['e2e']['ms_per_step'], d['speedup_vs_dense_sdpa'], d['roofline']['frac'], {k: round(v,2) for k,v in d['stages_ms'].items()})"; }
run "tpr2 wan"
run "tpr2 hunyuan" "--workload hunyuan-720p"
SVGEAR_ATTEND_TPR=1 run "tpr1 wan"
