# One C5 view (OBOX, gs_render): ncu --set full with source counters on every kernel of the
# frame (preprocess, the binning chain, the blend), then the per-kernel summary and the
# blend's per-source-line counters. Usage: bash tools/profile_job.sh TAG
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-prof}
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 ncu --set full --import-source on --clock-control none -c 40 -f -o gpurun_out/$TAG \
  python tools/profile_frame.py --obox --frames 1 > gpurun_out/${TAG}_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/$TAG.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source cuda -k regex:k_blend_tc > gpurun_out/${TAG}_blend_src.csv 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass -k regex:k_blend_tc > gpurun_out/${TAG}_blend_sass.csv 2>&1
ls -la gpurun_out/
