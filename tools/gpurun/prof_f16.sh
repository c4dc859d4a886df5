# ncu --set full of one f16 VGG-CIFAR stack pass (config 4, launches from the bench's f16 line)
mkdir -p gpurun_out
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_direct|k_dimg|k_lane|k_transpose" -s 13 -c 13 \
   -o /tmp/prof_f16 python tools/profile_stack.py --f16 --launches profiles/r02_launches_f16.json --passes 2 > gpurun_out/ncu_f16.log 2>&1
ncu -i /tmp/prof_f16.ncu-rep --page raw --csv > gpurun_out/ncu_f16_raw.csv 2>> gpurun_out/ncu_f16.log
echo done
