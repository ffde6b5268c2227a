# stale-threshold compositor + packed tile header: GPU suite, A/B sweep, preprocess (group 16) capture
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x > gpurun_out/r2_gpu_tests_m2.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_m2.txt
timeout 1500 python tools/sweep_blend.py --run --variants "stale1:;stale0:GS_BLEND_STALE_THR=0;raw1:GS_BLEND_RAW=1;stale1b:;stale0b:GS_BLEND_STALE_THR=0" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-configs" > gpurun_out/r2_sweep_m.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_preprocess -c 1 -f -o gpurun_out/r2_prof_pre16m python tools/profile_frame.py --obox --frames 1 --group 16 > gpurun_out/r2_prof_pre16m.log 2>&1
