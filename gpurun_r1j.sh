mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --launches gpurun_out/launches_vgg5.json > gpurun_out/bench.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu --no-dense --no-f16 --launches gpurun_out/launches_vgg5.json > gpurun_out/bench_torchrun.log 2>&1
timeout 1500 python tools/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
echo done
