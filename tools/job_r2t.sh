# L2 prefetch of the blend's record gathers: GPU suite, A/B sweep
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2_gpu_tests_t.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_t.txt
timeout 1800 python tools/sweep_blend.py --run --variants "pf1:;pf0:GS_BLEND_L2PF=0;pf2:GS_BLEND_L2PF=2;pf1r2:GS_BLEND_RAW=2;pf2r2:GS_BLEND_L2PF=2,GS_BLEND_RAW=2;pf1b:;pf0b:GS_BLEND_L2PF=0" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_t.txt 2>&1
