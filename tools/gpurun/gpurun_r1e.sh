mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python tools/probe_vgg.py > gpurun_out/probe.log 2>&1
echo done
