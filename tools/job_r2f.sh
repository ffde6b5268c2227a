set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q --timeout 60 -k "tc_color" > gpurun_out/r2_gpu_tests_h0.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_h0.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2_gpu_tests_h.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_h.txt
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-sweep --no-configs > gpurun_out/r2_bench_h.json 2> gpurun_out/r2_bench_h.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_preprocess -c 1 -f -o gpurun_out/r2_prof_pre16 python tools/profile_frame.py --obox --frames 1 --group 16 > gpurun_out/r2_prof_pre16.log 2>&1
