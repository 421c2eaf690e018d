# Round evidence in one call: tests, smoke, bench lines (2DSW + SOR), reference
# arms, the ncu launch list of the default bench command, ncu --set full of the
# default step kernel.  usage: bash tools/gpu_evidence.sh <label>
label=${1:-r01}
mkdir -p gpurun_out/ev_$label
D=gpurun_out/ev_$label
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $D/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf > $D/gpu_tests.log 2>&1; tail -2 $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; tail -2 $D/smoke.log
timeout 900 python bench.py > $D/bench.jsonl 2> $D/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $D/bench_reference.jsonl 2> $D/bench_reference.err; echo "ref rc=$?"
for w in "--workload c3" "--workload c5 --reduce none" "--workload c5 --reduce all" "--workload c2 --substeps 10000" "--workload c2 --substeps 10000 --reduce volume" "--workload p1000 --substeps 10000" "--workload p2000 --substeps 1000" "--workload c1 --substeps 1000" "--variant paper --steps 3" "--workload sor300" "--workload sor300 --sor-residual-every 0" "--workload sor1024 --steps 5"; do
  timeout 900 python bench.py --no-cpu-baseline $w >> $D/bench_more.jsonl 2>> $D/bench_more.err
done
SW2D_TWO_STEP=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e >> $D/bench_more.jsonl 2>> $D/bench_more.err
timeout 600 python bench.py --workload sor300 --impl reference --steps 3 --warmup 1 >> $D/bench_more.jsonl 2>> $D/bench_more.err
C="python bench.py --steps 2 --warmup 3"
timeout 900 $C > $D/plain_launch.log 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $D/launches.csv $C > $D/ncu_launch.log 2>&1
echo "launch list rc=$?"
Q="python bench.py --profile --steps 1 --warmup 3 --substeps 4"
timeout 600 $Q > $D/plain_prof.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sw2d_step -s 4 -c 1 -o $D/prof_c5 $Q > $D/ncu_prof.log 2>&1
python tools/ncu_summary.py $D/prof_c5.ncu-rep ${label}_c5 --cells 268435456 > $D/ncu_c5.json 2>&1; echo "prof rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sw2d_step -s 4 -c 1 -o $D/prof_c3 $Q --workload c3 > $D/ncu_prof_c3.log 2>&1
python tools/ncu_summary.py $D/prof_c3.ncu-rep ${label}_c3 --cells 67108864 > $D/ncu_c3.json 2>&1; echo "prof c3 rc=$?"
python - <<P
import json
for f in ["$D/bench.jsonl","$D/bench_reference.jsonl","$D/bench_more.jsonl"]:
    for l in open(f):
        try: d=json.loads(l)
        except Exception: continue
        r=d.get("roofline") or {}; e=d.get("e2e") or {}
        print(d.get("impl","ours"), d["config"]["workload"][:10], "%.3e"%d["value"], "ms/step %.3f"%d["ms_per_step"], "frac", r.get("frac"), r.get("bound"), "e2e %.3e"%(e.get("value") or 0), "launches", d.get("gpu_launches"), (d.get("clocks") or {}).get("sm_mhz"))
P
