set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/probe_vgg.py > gpurun_out/probe.log 2>&1
echo done
