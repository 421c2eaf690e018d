# Round evidence in one call: tests, smoke, bench lines (2DSW + SOR), reference
# arms, A/B of the small-grid kernels, the ncu launch list of the default
# bench command, ncu --set full of the step kernels.
#   usage: bash tools/gpu_evidence.sh <label>
label=${1:-r02}
mkdir -p gpurun_out/ev_$label
D=gpurun_out/ev_$label
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > $D/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $D/gpu_tests.log 2>&1; tail -2 $D/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; tail -3 $D/smoke.log
timeout 900 python bench.py > $D/bench.jsonl 2> $D/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > $D/bench_reference.jsonl 2> $D/bench_reference.err; echo "ref rc=$?"
for w in "--workload c3" "--workload c5 --reduce none" "--workload c5 --reduce all" "--workload c4 --steps 3 --no-e2e" "--workload c2" "--workload c2 --reduce volume" "--workload c2 --reduce all" "--workload p1000" "--workload p2000 --substeps 1000" "--workload c1 --substeps 1000" "--workload c1 --substeps 1000 --reduce all" "--variant paper --steps 3" "--snapshots --no-e2e" "--workload sor300" "--workload sor300 --sor-residual-every 0" "--workload sor1024 --steps 5" "--workload sor1024 --steps 5 --sor-residual-every 0"; do
  timeout 900 python bench.py --no-cpu-baseline $w >> $D/bench_more.jsonl 2>> $D/bench_more.err
done
SW2D_TWO_STEP=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e >> $D/bench_more.jsonl 2>> $D/bench_more.err
SW2D_FORCE_NCCL=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e >> $D/bench_more.jsonl 2>> $D/bench_more.err
SW2D_FORCE_NCCL=1 timeout 900 python bench.py --no-cpu-baseline --no-e2e --halo p2p >> $D/bench_more.jsonl 2>> $D/bench_more.err
timeout 600 python bench.py --workload sor300 --impl reference --steps 3 --warmup 1 >> $D/bench_more.jsonl 2>> $D/bench_more.err
bash tools/ab_env.sh ${label}_small "SW2D_PERSIST=0;SW2D_PERSIST=1" "--workload c2|--workload c2 --reduce volume|--workload c1 --substeps 1000|--workload c1 --substeps 1000 --reduce volume" 1 > /dev/null
cp gpurun_out/ab_${label}_small.log $D/ab_small.log
C="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 $C > $D/plain_launch.log 2>&1 && \
  timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $D/launches.csv $C > $D/ncu_launch.log 2>&1
echo "launch list rc=$?"
Q="python bench.py --profile --steps 1 --warmup 3 --substeps 4"
timeout 600 $Q > $D/plain_prof.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sw2d_step -s 4 -c 1 -o $D/prof_c5 $Q > $D/ncu_prof.log 2>&1
python tools/ncu_summary.py $D/prof_c5.ncu-rep ${label}_c5 > $D/ncu_c5.json 2>&1; echo "prof rc=$?"
timeout 600 $Q --workload c3 > $D/plain_prof_c3.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sw2d_step -s 4 -c 1 -o $D/prof_c3 $Q --workload c3 > $D/ncu_prof_c3.log 2>&1
python tools/ncu_summary.py $D/prof_c3.ncu-rep ${label}_c3 > $D/ncu_c3.json 2>&1; echo "prof c3 rc=$?"
P2="python bench.py --workload c2 --profile --steps 1 --warmup 1 --substeps 200"
timeout 300 $P2 > $D/plain_prof_c2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:persist -c 1 -o $D/prof_c2 $P2 > $D/ncu_prof_c2.log 2>&1
python tools/ncu_summary.py $D/prof_c2.ncu-rep ${label}_c2 > $D/ncu_c2.json 2>&1; echo "prof c2 rc=$?"
S="python bench.py --workload sor300 --profile --steps 1 --warmup 1"
timeout 300 $S > $D/plain_prof_sor.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sor_iter -s 3 -c 1 -o $D/prof_sor300 $S > $D/ncu_prof_sor.log 2>&1
python tools/ncu_summary.py $D/prof_sor300.ncu-rep ${label}_sor300 > $D/ncu_sor300.json 2>&1; echo "prof sor rc=$?"
python - <<P
import json
for f in ["$D/bench.jsonl","$D/bench_reference.jsonl","$D/bench_more.jsonl"]:
    for l in open(f):
        try: d=json.loads(l)
        except Exception: continue
        r=d.get("roofline") or {}; e=d.get("e2e") or {}
        print(d.get("impl","ours"), d["config"]["workload"][:10], "%.3e"%d["value"], "ms/step %.3f"%d["ms_per_step"], "frac", r.get("frac"), r.get("bound"), "e2e %.3e"%(e.get("value") or 0), "launches", d.get("gpu_launches"), (d.get("clocks") or {}).get("sm_mhz"), (r.get("plan") or "")[:50])
P
cat $D/ab_small.log
