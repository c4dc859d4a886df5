# ncu launch list + --set full capture of one VGG-CIFAR stack pass (13 kernels: the layout
# changes are fused into the neighbouring layers) with launches from the bench's line
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python tools/profile_stack.py --launches profiles/r02_launches_vgg_v12.json --passes 2 > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_direct|k_plane|k_dimg|k_dws|k_tiled|k_dtm|k_lane|k_transpose" -s 13 -c 13 \
   -o /tmp/prof_stack python tools/profile_stack.py --launches profiles/r02_launches_vgg_v12.json --passes 2 > gpurun_out/ncu_full.log 2>&1
ncu -i /tmp/prof_stack.ncu-rep --page raw --csv > gpurun_out/ncu_full_raw.csv 2>> gpurun_out/ncu_full.log
echo done
