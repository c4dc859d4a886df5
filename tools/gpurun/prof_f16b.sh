mkdir -p gpurun_out
for cfg in "conv2_2 395,16,4,8,16,16,2" "conv4_2 251,8,32,4,4,32,0"; do
  set -- $cfg
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_direct|k_plane" -s 2 -c 1 -o /tmp/h_$1 python tools/profile_one.py $1 $2 f16 > gpurun_out/h_$1.log 2>&1
  ncu -i /tmp/h_$1.ncu-rep --page raw --csv > gpurun_out/h_$1_raw.csv 2>>gpurun_out/h_$1.log
  ncu -i /tmp/h_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/h_$1_sass.csv 2>>gpurun_out/h_$1.log
done
