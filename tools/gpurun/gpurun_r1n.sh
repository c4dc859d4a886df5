mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 120 -p no:cacheprovider -k "direct_kernels_bitwise" > gpurun_out/pytest_tm.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_tm.log
timeout 900 python tools/probe_vgg.py > gpurun_out/probe.log 2>&1
echo done
