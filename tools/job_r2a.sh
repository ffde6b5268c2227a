set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_v3.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v3.txt
timeout 1200 python tools/sweep_blend.py --run --variants "bulk:;ldgsts:GS_BLEND_BULK=0;bulkb:;ldgstsb:GS_BLEND_BULK=0" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_bulk.txt 2>&1
bash tools/profile_job.sh r2_prof_v1
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool initcheck --error-exitcode 9 python tests/sanitize_cases.py --quick > gpurun_out/r2_sanitize_initcheck_v2.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitize_initcheck_v2.txt
timeout 900 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python tests/sanitize_cases.py --quick > gpurun_out/r2_sanitize_racecheck_v2.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_sanitize_racecheck_v2.txt
