# binning chains one stream priority above the preprocess, repeated
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python tools/sweep_blend.py --run --variants "p0:;p1:GS_CHAIN_PRIO=1;p0b:;p1b:GS_CHAIN_PRIO=1;p0c:;p1c:GS_CHAIN_PRIO=1" --bench-args "--steps 20 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_ae.txt 2>&1
