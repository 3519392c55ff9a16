import numpy as np, torch, sys
sys.path.insert(0,'.')
from paper_2405_10923_b200 import workloads as wl
W = wl.illcond_w(1<<20,128,7)
s = np.linalg.svd(W, compute_uv=False); ref = s[0]/s[-1]
Wd = torch.from_numpy(np.asfortranarray(W)).cuda()
R = torch.linalg.qr(Wd, mode="r")[1]
out = {}
for drv in (None, "gesvd", "gesvdj", "gesvda"):
    try:
        v = torch.linalg.svdvals(R, driver=drv); out[str(drv)] = float(v[0]/v[-1])
    except Exception as e: out[str(drv)] = repr(e)[:80]
sv = np.linalg.svd(R.cpu().numpy(), compute_uv=False); out["host_svd_of_devR"] = sv[0]/sv[-1]
Rn = np.linalg.qr(W, mode="r"); sv = np.linalg.svd(Rn, compute_uv=False); out["numpy_qr_svd"] = sv[0]/sv[-1]
for k, v in out.items():
    print(k, v, (v-ref)/ref if isinstance(v, float) else "")
print("ref", ref)
