"""Phase split of the reduce kernel on c2 (values pass)."""
import json, sys
import torch
sys.path.insert(0, ".")
import paper_2605_16058_b200 as sb
from paper_2605_16058_b200 import _native as nat
from paper_2605_16058_b200.configs import config2
from paper_2605_16058_b200.mode_product import forward_device
from paper_2605_16058_b200.slice_svd import svd_values_device
a = config2(nlat=361, nlon=720, nt=1024, seed=0)
ts = sb.TransformSet.build(a.shape, "dct")
x = sb.DeviceTensor.from_host(sb.DenseTensor(a, copy=False), torch.device("cuda", 0))
ah = sb.DeviceTensor(forward_device(x, ts).data, a.shape)
lib = nat.load()
lib.starm_svd_tune(-1, -1, -1, 1)
svd_values_device(ah); torch.cuda.synchronize(); nat.svd_stats(reset=True)
svd_values_device(ah); torch.cuda.synchronize()
st = nat.svd_stats(reset=True)
n = st["slices"] or 1024
per = {k: round(v / 1024 / 1e6, 3) for k, v in st.items() if k.startswith("cyc_")}
print(json.dumps({"Mcycles_per_slice": per}))
