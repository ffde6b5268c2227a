set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_g.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_f.txt
timeout 1200 python tools/sweep_blend.py --run --variants "base:;base2:" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_g.txt 2>&1
bash tools/profile_job.sh r2_prof_v8
