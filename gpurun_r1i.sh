mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/prof_c32_jump python tools_profile_layer.py --layer conv3_2 --reps 1 --launch 14,8,4,8,8,16 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/prof_c32_mask python tools_profile_layer.py --layer conv3_2 --reps 1 --launch 15,8,4,8,8,16 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/prof_c51 python tools_profile_layer.py --layer conv5_1 --reps 1 --launch 14,4,32,2,4,8 > gpurun_out/ncu3.log 2>&1
timeout 900 python tools_debug_variants.py > gpurun_out/debug_variants.log 2>&1
echo done
