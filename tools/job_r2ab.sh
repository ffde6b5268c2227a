# OBOX lim once per Gaussian: GPU suite, two bench runs, preprocess capture
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2_gpu_tests_ab.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_ab.txt
for i in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["stage_ms_per_frame"])' >> gpurun_out/r2_sweep_ab.txt; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_preprocess -c 1 -f -o gpurun_out/r2_prof_pre16ab python tools/profile_frame.py --obox --frames 1 --group 16 > gpurun_out/r2_prof_pre16ab.log 2>&1
