run() { python bench.py --no-sweep --no-dense --no-cpu-baseline --steps 5 --warmup 3 $2 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['ms_per_step'], d['e2e']['ms_per_step'], d['config']['kmeans_iters_run'], {k: round(v,2) for k,v in d['stages_ms'].items()}, d['config']['rel_l2_vs_dense_head0'])"; }
run "quad"
tools/rebuild_with.sh seed.cu "-DSVG_SEED_T8=853 -DSVG_SEED_T4=426 -DSVG_SEED_T2=106"; run "T853/426/106"
tools/rebuild_with.sh seed.cu "-DSVG_SEED_T8=853 -DSVG_SEED_T4=426 -DSVG_SEED_T2=106 -DSVG_SEED_GREEDY=150"; run "T853/426/106 g150"
tools/rebuild_with.sh seed.cu "-DSVG_SEED_T8=10000 -DSVG_SEED_T4=10000 -DSVG_SEED_T2=10000 -DSVG_SEED_GREEDY=150"; run "all single g150"
