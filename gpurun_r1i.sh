mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -p no:cacheprovider -k "f16 or direct or image_lane" > gpurun_out/pytest_direct.log 2>&1
timeout 900 python gpurun_probe.py > gpurun_out/probe.log 2>&1
timeout 900 python tools/sweep.py --out gpurun_out/sweep.json --sparsities 0.5,0.9,0.99 > gpurun_out/sweep.log 2>&1
echo done
