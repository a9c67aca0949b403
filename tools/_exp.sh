run() { echo "$1: $(env $1 python bench.py --no-sweep --no-dense --no-cpu-baseline --steps 5 --warmup 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'])")"; }
run A=0
run SVGEAR_GROUP_FRACTIONS=0.3,1.0
run SVGEAR_GROUP_FRACTIONS=0.4,1.0
run SVGEAR_GROUP_FRACTIONS=0.2,1.0
run SVGEAR_GROUP_FRACTIONS=0.7,1.0
run SVGEAR_ATTEND_G=2
