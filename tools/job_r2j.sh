set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2_gpu_tests_l.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_l.txt
timeout 1500 python bench.py > gpurun_out/r2_bench_l.json 2> gpurun_out/r2_bench_l.err
bash tools/profile_job.sh r2_prof_v10
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2_launches_l.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs > gpurun_out/r2_launches_l.log 2>&1
