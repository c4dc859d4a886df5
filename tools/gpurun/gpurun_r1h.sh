mkdir -p gpurun_out
timeout 900 python bench.py --launches gpurun_out/launches_vgg4.json > gpurun_out/bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_direct|k_plane|k_dimg" -s 14 -c 13 \
   -o gpurun_out/prof_stack4 python tools/profile_stack.py --launches gpurun_out/launches_vgg4.json --passes 2 > gpurun_out/ncu_full.log 2>&1
echo done
