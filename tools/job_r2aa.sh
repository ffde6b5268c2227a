# per-half TMEM-stage / named barriers in the tcgen05 blend (GS_BLEND_HALVES): parity suite on that build, A/B sweep
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
GS_RENDER_LIB=$GRAFT_REPO_ROOT/paper_2604_02120_b200/variants/lib_h1.so timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_h1.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke_h1.txt
if grep -q "rc=0" gpurun_out/r2_smoke_h1.txt; then
GS_RENDER_LIB=$GRAFT_REPO_ROOT/paper_2604_02120_b200/variants/lib_h1.so timeout 900 python -m pytest tests -m gpu -q -x --timeout 120 > gpurun_out/r2_gpu_tests_h1.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_h1.txt
timeout 1500 python tools/sweep_blend.py --run --variants "h0:;h1:GS_BLEND_HALVES=1;h0b:;h1b:GS_BLEND_HALVES=1" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-configs" > gpurun_out/r2_sweep_aa.txt 2>&1
fi
