mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/prof_conv3_2_v2 python tools_profile_layer.py --layer conv3_2 --reps 1 --launch 0,4,16,8,8,16 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/prof_conv1_2_v2 python tools_profile_layer.py --layer conv1_2 --reps 1 --launch 14,1,1,32,32,8 > gpurun_out/ncu2.log 2>&1
echo done
