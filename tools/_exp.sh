run() { python bench.py --no-sweep --no-dense --no-cpu-baseline --steps 5 --warmup 3 $2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['e2e']['ms_per_step'], d['config']['kmeans_iters_run'], {k: round(v,2) for k,v in d['stages_ms'].items()}, d['config']['rel_l2_vs_dense_head0'])"; }
python tools/seed_time.py 2>&1 | grep -E "key_side|seed_gram"
run "filter"
run "filter hunyuan" "--workload hunyuan-720p"
tools/rebuild_with.sh seed.cu "-DSVG_SEED_FILTER=0"; run "nofilter"
