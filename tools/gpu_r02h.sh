set -x
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/r02h_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02h_gpu_tests.log
tail -3 gpurun_out/r02h_gpu_tests.log
grep -q "rc=0" gpurun_out/r02h_gpu_tests.log || exit 1
P=paper_1711_04471_b200
bash tools/ab_libs.sh r02h "$P/libsw2d_prev.so $P/libsw2d.so $P/libsw2d_enonly.so" "--workload c5|--workload c5 --reduce none|--workload c3|--workload c5 --reduce all|--workload p2000" 2
Q="python bench.py --workload c2 --profile --steps 1 --warmup 1 --substeps 200"
SW2D_PERSIST=1 timeout 300 $Q > gpurun_out/plain_r02h_persist.log 2>&1 && \
  SW2D_PERSIST=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:persist -c 1 -o gpurun_out/prof_r02h_persist $Q > gpurun_out/ncu_r02h_persist.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_r02h_persist.ncu-rep r02h_persist > gpurun_out/summary_r02h_persist.json 2>&1; head -30 gpurun_out/summary_r02h_persist.json
