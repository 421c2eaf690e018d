mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/gpu_all_tests.log 2>&1; tail -3 gpurun_out/gpu_all_tests.log
rm -f gpurun_out/r01_sor_bench.jsonl
timeout 300 python bench.py --workload sor300 --steps 10 --warmup 3 >> gpurun_out/r01_sor_bench.jsonl 2> gpurun_out/bench_sor300.err
timeout 300 python bench.py --workload sor300 --steps 10 --warmup 3 --sor-residual-every 0 --no-cpu-baseline >> gpurun_out/r01_sor_bench.jsonl 2>> gpurun_out/bench_sor300.err
timeout 300 python bench.py --workload sor1024 --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/r01_sor_bench.jsonl 2> gpurun_out/bench_sor1024.err
timeout 300 python bench.py --workload sor300 --impl reference --steps 3 --warmup 1 >> gpurun_out/r01_sor_bench.jsonl 2>> gpurun_out/bench_sor300.err
python - <<'P'
import json
for l in open("gpurun_out/r01_sor_bench.jsonl"):
    d=json.loads(l); r=d.get("roofline") or {}; e=d.get("e2e") or {}
    print(d.get("impl","ours"), d["config"]["workload"][:8], d["config"].get("residual_every"), "%.3e"%d["value"], "frac", r.get("frac"), "traffic", r.get("traffic"), "e2e %.3e"%e.get("value",0), d.get("gpu_launches"), d.get("clocks"))
P
