mkdir -p gpurun_out
timeout 900 python tools_debug_variants.py > gpurun_out/debug_variants.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python gpurun_probe.py > gpurun_out/probe.log 2>&1
echo done
