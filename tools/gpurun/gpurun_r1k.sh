mkdir -p gpurun_out
python - <<'PY'
import json
json.dump([[16, 8, 1, 8, 32, 4, 2], [10, 8, 1, 8, 32, 16, 2], [85, 8, 2, 8, 16, 16, 2], [85, 8, 2, 8, 16, 16, 2], [12, 8, 4, 8, 8, 16, 2], [12, 8, 4, 8, 8, 16, 2], [12, 8, 4, 8, 8, 16, 2], [156, 8, 32, 4, 4, 16, 0], [156, 8, 32, 4, 4, 16, 0], [156, 8, 32, 4, 4, 16, 0], [72, 8, 32, 2, 2, 32, 2], [72, 8, 32, 2, 2, 32, 2], [72, 8, 32, 2, 2, 32, 2]], open("gpurun_out/launches_cur.json","w"))
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_direct|k_plane|k_dimg" -s 13 -c 13 \
   -o gpurun_out/prof_stack5 python tools/profile_stack.py --launches gpurun_out/launches_cur.json --passes 2 > gpurun_out/ncu_full.log 2>&1
echo done
