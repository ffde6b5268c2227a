set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "preprocess or view_groups or random or scale_modifier or C5 or obox_pre or C1 or C2 or ragged or dense" > gpurun_out/r2_gpu_tests_k.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_k.txt
timeout 1500 python tools/sweep_blend.py --run --variants "base:;nocompact:GS_PRE_COMPACT=0;nol1pf:GS_BLEND_L1PF=0;notma:GS_BLEND_TMA_STORE=0;lpf2h0:GS_BLEND_LPF=2,GS_BLEND_HPF=0;base2:" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_k.txt 2>&1
