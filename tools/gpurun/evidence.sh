mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 1200 python bench.py --launches gpurun_out/launches_vgg.json > gpurun_out/bench.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python tools/profile_stack.py --launches gpurun_out/launches_vgg.json --passes 2 > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"k_direct|k_plane|k_dimg|k_dws|k_tiled|k_dtm|k_lane|k_tile|k_transpose" -s 14 -c 14 \
   -o /tmp/prof_stack python tools/profile_stack.py --launches gpurun_out/launches_vgg.json --passes 2 > gpurun_out/ncu_full.log 2>&1
# the full report exceeds gpurun's 64 MiB return limit: bring back its raw page as CSV
ncu -i /tmp/prof_stack.ncu-rep --page raw --csv > gpurun_out/ncu_full_raw.csv 2>> gpurun_out/ncu_full.log
echo done
