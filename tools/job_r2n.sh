# compacted view-group preprocess: GPU suite (+ the RAW=1 blend variant's suite), A/B sweep
set -x
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2_gpu_tests_n.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_n.txt
GS_RENDER_LIB=$GRAFT_REPO_ROOT/paper_2604_02120_b200/variants/lib_raw1c.so timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r2_gpu_tests_n_raw1.txt 2>&1; echo "rc=$?" >> gpurun_out/r2_gpu_tests_n_raw1.txt
timeout 1500 python tools/sweep_blend.py --run --variants "cv1:;cv0:GS_PRE_CV=0;raw1c:GS_BLEND_RAW=1;cv1b:;cv0b:GS_PRE_CV=0;raw1cb:GS_BLEND_RAW=1" --bench-args "--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-ab --no-sweep --no-configs" > gpurun_out/r2_sweep_n.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_preprocess -c 1 -f -o gpurun_out/r2_prof_pre16n python tools/profile_frame.py --obox --frames 1 --group 16 > gpurun_out/r2_prof_pre16n.log 2>&1
