set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gpu_tests_v2.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_gpu_tests_v2.txt
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 9 python tests/sanitize_cases.py > gpurun_out/r2_sanitize_$tool.txt 2>&1
  echo "compute-sanitizer $tool rc=$?" >> gpurun_out/r2_sanitize_$tool.txt
done
timeout 1500 $CS --tool racecheck --racecheck-report all --error-exitcode 9 python tests/sanitize_cases.py --quick > gpurun_out/r2_sanitize_racecheck.txt 2>&1
echo "compute-sanitizer racecheck rc=$?" >> gpurun_out/r2_sanitize_racecheck.txt
tail -3 gpurun_out/r2_sanitize_*.txt
