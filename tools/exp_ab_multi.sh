# A/B/.. of library builds on one bench line: bash tools/exp_ab_multi.sh "bench args" lib1 lib2 ...
args=$1; shift
for r in 1 2; do for lib in "$@"; do
  SW2D_LIBRARY=paper_1711_04471_b200/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $args 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '%.4e'%d['value'], d['clocks']['sm_mhz'])"
done; done
