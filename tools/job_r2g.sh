set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 120 -k "C1 or ragged or C2 or dense or adversarial" > gpurun_out/r2_gpu_tests_i.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_i.txt
timeout 900 python tools/sweep_blend.py --run --variants "base:;base2:" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_i.txt 2>&1
bash tools/profile_job.sh r2_prof_v9
