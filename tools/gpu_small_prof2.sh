C="python bench.py --workload c2 --substeps 16 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --profile"
timeout 300 $C > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:sw2d_step_small -s 8 -c 1 -o gpurun_out/prof_small $C > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/prof_small.ncu-rep small --cells 250000 | head -45
ncu -i gpurun_out/prof_small.ncu-rep --page details --csv 2>/dev/null | grep -iE "Duration|Elapsed Cycles|SM Active Cycles|Achieved Occupancy|Theoretical Occupancy|Waves Per SM|Registers|Block Limit" | head -20
