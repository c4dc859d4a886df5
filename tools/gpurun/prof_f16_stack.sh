# ncu --set full of one f16-storage (config 4) VGG-CIFAR pass with tuned launches; raw page as CSV
mkdir -p gpurun_out
python - <<'PY'
import json, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2011_06295_b200.network import build_net
from paper_2011_06295_b200.synth import vgg16_cifar
net = build_net(vgg16_cifar(0.9), dtype=np.float16)
net.plan(256, tune=True)
json.dump([None if l is None else list(l) for l in net.launches], open("gpurun_out/launches_f16.json", "w"))
PY
timeout 900 ncu -f --set full --clock-control none -k regex:"k_direct|k_plane|k_dimg|k_tiled" -s 13 -c 13 \
   -o /tmp/prof_f16 python tools/profile_stack.py --f16 --launches gpurun_out/launches_f16.json --passes 2 \
   > gpurun_out/ncu_f16.log 2>&1
ncu -i /tmp/prof_f16.ncu-rep --page raw --csv > gpurun_out/ncu_f16_raw.csv 2>> gpurun_out/ncu_f16.log
