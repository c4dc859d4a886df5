"""Per-layer DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum, bytes
per launch) of one profiled forward pass of the VGG-CIFAR stack -> JSON
{layer: bytes} for bench.py's roofline.traffic.  Usage:
  python tools/traffic_from_ncu.py <report.ncu-rep | raw-page.csv> <launches.json> > profiles/traffic.json
Conv launches are matched to layers in order; a generic layer with a fused
pool contributes its conv launch plus the following k_maxpool2 launch."""
import csv
import io
import json
import subprocess
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
from paper_2011_06295_b200.synth import vgg16_cifar  # noqa: E402

rep, lf = sys.argv[1], sys.argv[2]
launches = json.load(open(lf))
raw = open(rep).read() if rep.endswith(".csv") else \
    subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
iN, iR, iW = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
units = r[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rows = [(x[iN], float(x[iR]) * scale[units[iR]] + float(x[iW]) * scale[units[iW]]) for x in r[2:]]
rows = [x for x in rows if "k_transpose" not in x[0]]  # layout conversions are not a layer's kernel
# drop leading pool launches that belong to the previous pass
while rows and "maxpool" in rows[0][0]:
    rows.pop(0)
out = {}
i = 0
for (spec, pool), l in zip(vgg16_cifar(0.9), launches):
    if i >= len(rows):
        break
    b = rows[i][1]
    i += 1
    if l is None and pool and i < len(rows) and "maxpool" in rows[i][0]:
        b += rows[i][1]
        i += 1
    out[spec.name] = int(b)
print(json.dumps(out, indent=1))
