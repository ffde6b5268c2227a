cd $GRAFT_REPO_ROOT
python -c "
import torch,os
pr=torch.cuda.get_device_properties(0); print(pr); print([a for a in dir(pr) if 'pci' in a])
import bench
print('local', sorted(bench._gpu_local_cpus(0) or [])[:8], len(bench._gpu_local_cpus(0) or []), 'of', len(os.sched_getaffinity(0)))
" > gpurun_out/r2_numa_probe.txt 2>&1
nvidia-smi topo -m >> gpurun_out/r2_numa_probe.txt 2>&1
python tools/pcie_probe.py >> gpurun_out/r2_numa_probe.txt 2>&1
python -c "
import os,bench; c=bench._gpu_local_cpus(0); os.sched_setaffinity(0,c) if c else None
import runpy; runpy.run_path('tools/pcie_probe.py')" >> gpurun_out/r2_numa_probe.txt 2>&1
timeout 900 python bench.py --no-ab --no-sweep --no-configs --no-cpu-baseline > gpurun_out/r2_bench_z.json 2> gpurun_out/r2_bench_z.err
