set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -k "identically" > gpurun_out/r2_gpu_tests_m.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_m.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-configs > gpurun_out/r2_bench_m.json 2> gpurun_out/r2_bench_m.err
bash tools/sanitize_job.sh
