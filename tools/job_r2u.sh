# helper warps polling with a sleep between tries: A/B sweep (+ one ncu capture of the 256-ns variant)
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python tools/sweep_blend.py --run --variants "sl0:;sl64:GS_HELPER_SLEEP_NS=64;sl256:GS_HELPER_SLEEP_NS=256;sl1000:GS_HELPER_SLEEP_NS=1000;sl0b:" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_u.txt 2>&1
GS_RENDER_LIB=$GRAFT_REPO_ROOT/paper_2604_02120_b200/variants/lib_sl256.so timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_blend_tc -c 1 -f -o gpurun_out/r2_prof_u python tools/profile_frame.py --obox --frames 1 > gpurun_out/r2_prof_u.log 2>&1
