# A/B of two library builds on the C5 bench line: bash tools/exp_ab_c5.sh libA libB [bench args]
a=$1; b=$2; shift 2
for r in 1 2; do for lib in $a $b; do
  SW2D_LIBRARY=paper_1711_04471_b200/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '%.4e'%d['value'], d['clocks'])"
done; done
