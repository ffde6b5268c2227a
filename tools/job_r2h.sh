set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "preprocess or view_groups or random or scale_modifier or C5 or obox_pre" > gpurun_out/r2_gpu_tests_j.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_j.txt
timeout 1200 python tools/sweep_blend.py --run --variants "base:;nocompact:GS_PRE_COMPACT=0;base2:;nocompact2:GS_PRE_COMPACT=0" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_j.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_preprocess -c 1 -f -o gpurun_out/r2_prof_pre16b python tools/profile_frame.py --obox --frames 1 --group 16 > gpurun_out/r2_prof_pre16b.log 2>&1
