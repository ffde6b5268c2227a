# HEAD re-verification: full GPU suite, smoke, default bench line, bench launch list, one-view full capture
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 1800 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2_gpu_tests_l.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_l.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke_l.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_smoke_l.txt
timeout 1200 python bench.py > gpurun_out/r2_bench_l.json 2> gpurun_out/r2_bench_l.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2_launches_bench_l.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs > gpurun_out/r2_launches_bench_l.log 2>&1
bash tools/profile_job.sh r2_prof_l
