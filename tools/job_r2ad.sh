# concurrent-chain binning grid multiple 2 vs 3, repeated
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python tools/sweep_blend.py --run --variants "g3:;g2:GS_GRID_MULT_CONCURRENT=2;g3b:;g2b:GS_GRID_MULT_CONCURRENT=2;g3c:;g2c:GS_GRID_MULT_CONCURRENT=2" --bench-args "--steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_ad.txt 2>&1
