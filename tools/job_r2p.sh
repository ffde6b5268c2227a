# SH rows read with 16-B loads (preprocess), two-pass compositor A/B
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2_gpu_tests_p.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_p.txt
timeout 1500 python tools/sweep_blend.py --run --variants "base:;twopass:GS_BLEND_TWO_PASS=1;base2:;twopass2:GS_BLEND_TWO_PASS=1" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_p.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_preprocess -c 1 -f -o gpurun_out/r2_prof_pre16p python tools/profile_frame.py --obox --frames 1 --group 16 > gpurun_out/r2_prof_pre16p.log 2>&1
