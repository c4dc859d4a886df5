mkdir -p gpurun_out
timeout 900 python tools_debug_variants.py > gpurun_out/debug_variants.log 2>&1
echo done
