mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k plane > gpurun_out/pytest_plane.log 2>&1
timeout 900 python tools/probe_vgg.py > gpurun_out/probe.log 2>&1
echo done
