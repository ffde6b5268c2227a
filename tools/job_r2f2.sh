# final verification of HEAD: GPU suite (parity log), smoke, default bench, reference arm
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
GS_PARITY_LOG=$GRAFT_REPO_ROOT/gpurun_out/r2_parity_f.jsonl timeout 1800 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2_gpu_tests_f.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_f.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_f.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke_f.txt
timeout 1200 python bench.py > gpurun_out/r2_bench_f.json 2> gpurun_out/r2_bench_f.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2_bench_ref_f.json 2> gpurun_out/r2_bench_ref_f.err
