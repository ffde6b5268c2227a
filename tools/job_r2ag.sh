# occupancy knobs with the final build (scan / scatter / preprocess bounds, chunk size)
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python tools/sweep_blend.py --run --variants "base:;scan8:GS_SCAN_MINB=8;pre3:GS_PRE_MINB=3;scat2:GS_SCATTER_MINB=2;items16:GS_SORT_ITEMS=16;base2:;scan4:GS_SCAN_MINB=4" --bench-args "--steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_ag.txt 2>&1
