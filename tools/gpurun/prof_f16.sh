mkdir -p gpurun_out
for cfg in "f16 395,8,4,8,16,8,2 f16" "f32 100,8,2,8,16,16,2"; do
  set -- $cfg
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_direct" -s 2 -c 1 -o /tmp/p_$1 python tools/profile_one.py conv2_2 $2 $3 > gpurun_out/p_$1.log 2>&1
  ncu -i /tmp/p_$1.ncu-rep --page raw --csv > gpurun_out/p_$1_raw.csv 2>>gpurun_out/p_$1.log
  ncu -i /tmp/p_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/p_$1_sass.csv 2>>gpurun_out/p_$1.log
  ncu -i /tmp/p_$1.ncu-rep --page details --csv > gpurun_out/p_$1_details.csv 2>>gpurun_out/p_$1.log
done
ls -la gpurun_out
