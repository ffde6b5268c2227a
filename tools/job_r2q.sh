# supertile pairs materialised by the offsets scan: GPU suite (+ the StLoader variant), A/B sweep, launch list
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2_gpu_tests_q.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_q.txt
timeout 1500 python tools/sweep_blend.py --run --variants "stmat1:;stmat0:GS_ST_MAT=0;stmat1b:;stmat0b:GS_ST_MAT=0" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_q.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_launches_q.csv python tools/profile_frame.py --obox --frames 1 > gpurun_out/r2_launches_q.log 2>&1
