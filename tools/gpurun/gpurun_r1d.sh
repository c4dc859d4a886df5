mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --launches gpurun_out/launches_vgg2.json > gpurun_out/bench.log 2>&1
echo done
