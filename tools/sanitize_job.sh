# compute-sanitizer over tests/sanitize_cases.py (every blend, both binnings, view group,
# host entry points); logs into gpurun_out/r2_sanitize_<tool>_${TAG}.txt
set -x
TAG=${1:-v3}
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 9 python tests/sanitize_cases.py > gpurun_out/r2_sanitize_${tool}_${TAG}.txt 2>&1
  echo "compute-sanitizer $tool rc=$?" >> gpurun_out/r2_sanitize_${tool}_${TAG}.txt
done
# racecheck: every kernel but k_blend_tc (its mbarrier-ordered raw ring is reported as potential
# WAR hazards: racecheck does not model mbarrier phases), then k_blend_tc alone, summarised
timeout 1500 $CS --tool racecheck --racecheck-report hazard --kernel-name-exclude kns=k_blend_tc --error-exitcode 9 python tests/sanitize_cases.py --quick > gpurun_out/r2_sanitize_racecheck_other_${TAG}.txt 2>&1
echo "compute-sanitizer racecheck (all but k_blend_tc) rc=$?" >> gpurun_out/r2_sanitize_racecheck_other_${TAG}.txt
timeout 1500 $CS --tool racecheck --racecheck-report analysis --kernel-name kns=k_blend_tc --print-limit 20 python tests/sanitize_cases.py --quick > gpurun_out/r2_sanitize_racecheck_blend_${TAG}.txt 2>&1
echo "compute-sanitizer racecheck (k_blend_tc) rc=$?" >> gpurun_out/r2_sanitize_racecheck_blend_${TAG}.txt
