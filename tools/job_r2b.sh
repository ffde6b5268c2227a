set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_v5.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v5.txt
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs > gpurun_out/r2_bench_v3_quick.json 2> gpurun_out/r2_bench_v3_quick.err
bash tools/profile_job.sh r2_prof_v3
