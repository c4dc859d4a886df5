mkdir -p gpurun_out
./tools/tma_test > gpurun_out/tma_test.log 2>&1
timeout 900 python tools_debug_variants.py > gpurun_out/debug_variants.log 2>&1
echo done
