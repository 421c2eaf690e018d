mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf -x > gpurun_out/gpu_all_tests.log 2>&1; tail -3 gpurun_out/gpu_all_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
for w in "--workload c2 --substeps 1000 --reduce volume" "--workload c2 --substeps 1000 --reduce all" "--workload c2 --substeps 1000" "--workload c1 --substeps 1000 --reduce all"; do
  bash tools/exp_ab_multi.sh "$w" libsw2d_prev.so libsw2d.so
done
