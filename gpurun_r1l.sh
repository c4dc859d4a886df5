mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 900 python bench.py --launches gpurun_out/launches_vgg7.json > gpurun_out/bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_direct|k_plane|k_dimg|k_dws|k_tiled" -s 13 -c 13 \
   -o gpurun_out/prof_stack7 python tools/profile_stack.py --launches gpurun_out/launches_vgg7.json --passes 2 > gpurun_out/ncu_full.log 2>&1
echo done
