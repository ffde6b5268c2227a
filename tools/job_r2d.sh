set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "C1 or ragged or dense or C2 or adversarial or tight or obox" > gpurun_out/r2_gpu_tests_e.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_d.txt
timeout 1200 python tools/sweep_blend.py --run --variants "base:;raw3:GS_BLEND_RAW=3;raw4:GS_BLEND_RAW=4;hpf0:GS_BLEND_HPF=0;base2:" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_raw_e.txt 2>&1
bash tools/profile_job.sh r2_prof_v6
