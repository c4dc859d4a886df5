mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --steps 100 --no-cpu --no-dense --no-f16 --no-alexnet --launches gpurun_out/launches_vgg7.json > gpurun_out/bench_pdl.log 2>&1
echo done
