# upper bound of the no-op 4th depth pass's cost (variant that never launches it; C5 has no wide depths)
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python tools/sweep_blend.py --run --variants "base:;skipw:GS_SKIP_WIDE=1;base2:;skipw2:GS_SKIP_WIDE=1" --bench-args "--steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_ah.txt 2>&1
