# blend per-batch trace (CTA 0) + knob sweep on the RAW=1 build
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python tools/trace_blend.py > gpurun_out/r2_trace_o.txt 2>&1
timeout 1500 python tools/sweep_blend.py --run --variants "base:;lpf2:GS_BLEND_LPF=2;susp0:GS_MBAR_SUSPEND_NS=0;base2:" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_o.txt 2>&1
