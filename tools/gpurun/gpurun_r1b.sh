set -x
mkdir -p gpurun_out
timeout 900 python bench.py --launches gpurun_out/launches_vgg.json > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python tools/profile_stack.py --launches gpurun_out/launches_vgg.json --passes 2 > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tiled|k_generic|k_maxpool" -s 14 -c 16 \
   -o gpurun_out/prof_stack python tools/profile_stack.py --launches gpurun_out/launches_vgg.json --passes 2 > gpurun_out/ncu_full.log 2>&1
echo done
