# final-build verification: full GPU suite, smoke, default bench line, bench launch list, one-view full capture
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2_gpu_tests_s.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_s.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_s.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke_s.txt
timeout 1200 python bench.py > gpurun_out/r2_bench_s.json 2> gpurun_out/r2_bench_s.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r2_bench_ref_s.json 2> gpurun_out/r2_bench_ref_s.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2_launches_bench_s.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs > gpurun_out/r2_launches_bench_s.log 2>&1
bash tools/profile_job.sh r2_prof_s
