# orbit knob sweep on the final build: binning grid sizes, scatter occupancy, view group 8 / 32, hardware queues
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
BA="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs"
V=$GRAFT_REPO_ROOT/paper_2604_02120_b200/variants
timeout 1500 python tools/sweep_blend.py --run --variants "base:;gmc3:GS_GRID_MULT_CONCURRENT=3;gmc6:GS_GRID_MULT_CONCURRENT=6;smin4:GS_SCATTER_MINB=4;base2:" --bench-args "$BA" > gpurun_out/r2_sweep_v.txt 2>&1
for g in 8 32; do
  L=$V/lib_base.so; [ $g = 32 ] && L=$V/lib_vg32.so
  echo "group $g: $(GS_RENDER_LIB=$L GS_BENCH_GROUP=$g timeout 600 python bench.py $BA 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["stage_ms_per_frame"])')" >> gpurun_out/r2_sweep_v.txt
done
for q in 16 32; do
  echo "connections $q: $(CUDA_DEVICE_MAX_CONNECTIONS=$q GS_RENDER_LIB=$V/lib_base.so timeout 600 python bench.py $BA 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), d["stage_ms_per_frame"])')" >> gpurun_out/r2_sweep_v.txt
done
