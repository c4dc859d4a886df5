mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 300 -p no:cacheprovider -k quantized > gpurun_out/pytest_quant.log 2>&1
timeout 300 python -c "
import sys, ctypes, json; sys.path.insert(0,'.')
from paper_2011_06295_b200 import _abi
names = ctypes.create_string_buffer(16*8); vals=(ctypes.c_double*8)(); cnt=ctypes.c_int32()
_abi.check(_abi.lib().scb_fma_peaks(0, names, vals, 8, ctypes.byref(cnt)))
print(json.dumps({names.raw[16*i:16*i+16].split(b'\0')[0].decode(): round(vals[i]/1e9,1) for i in range(cnt.value)}))
" > gpurun_out/peaks.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/prof_conv3_2 python tools_profile_layer.py --layer conv3_2 --reps 1 > gpurun_out/ncu_conv3_2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tiled -c 1 -o gpurun_out/prof_conv1_2 python tools_profile_layer.py --layer conv1_2 --reps 1 --launch 0,2,2,32,32,4 > gpurun_out/ncu_conv1_2.log 2>&1
echo done
