mkdir -p gpurun_out
timeout 1500 python tools/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
echo done
