# concurrent-chain binning grid multiple 3 / 2 vs 4, repeated
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python tools/sweep_blend.py --run --variants "base:;gmc3:GS_GRID_MULT_CONCURRENT=3;gmc2:GS_GRID_MULT_CONCURRENT=2;base2:;gmc3b:GS_GRID_MULT_CONCURRENT=3;base3:;gmc3c:GS_GRID_MULT_CONCURRENT=3" --bench-args "--steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_ac.txt 2>&1
