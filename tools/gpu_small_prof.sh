mkdir -p gpurun_out
C="python bench.py --workload c2 --substeps 16 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --profile"
timeout 300 $C > gpurun_out/sp_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sp_tb_launches.csv $C > /dev/null 2>&1
SW2D_TB=0 timeout 300 $C > gpurun_out/sp_plain0.log 2>&1 && SW2D_TB=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sp_notb_launches.csv $C > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sw2d_step_tb -s 2 -c 1 -o gpurun_out/prof_tb $C > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/sp_tb_launches.csv tb | head -20
python tools/launch_summary.py gpurun_out/sp_notb_launches.csv notb | head -20
python tools/ncu_summary.py gpurun_out/prof_tb.ncu-rep tb | head -40
