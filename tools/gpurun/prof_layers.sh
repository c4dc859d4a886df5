# ncu --set full of single VGG-CIFAR layers with explicit launches; raw + sass pages back as CSV
mkdir -p gpurun_out
while [ $# -ge 2 ]; do
  L=$1; C=$2; shift 2
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_direct|k_dimg" -s 2 -c 1 -o /tmp/p_$L python tools/profile_one.py $L $C > gpurun_out/p_$L.log 2>&1
  ncu -i /tmp/p_$L.ncu-rep --page raw --csv > gpurun_out/p_${L}_raw.csv 2>>gpurun_out/p_$L.log
  ncu -i /tmp/p_$L.ncu-rep --page source --csv --print-source sass > gpurun_out/p_${L}_sass.csv 2>>gpurun_out/p_$L.log
done
