import numpy as np, torch, sys
sys.path.insert(0, ".")
from paper_2605_24514_b200 import _lib
lib=_lib.load()
np.set_printoptions(precision=4, linewidth=150)
for s in (3, 5):
    rng=np.random.default_rng(s)
    c=rng.standard_normal((1,s,s)); c[0,-1,:]=0
    d=torch.tensor(c,device="cuda"); u=torch.empty_like(d); vt=torch.empty_like(d); sv=torch.empty((1,s),dtype=torch.float64,device="cuda")
    _lib.check(lib.isvd_core_svd(1,s,d.data_ptr(),u.data_ptr(),sv.data_ptr(),vt.data_ptr(),None))
    torch.cuda.synchronize()
    print(s, sv.cpu().numpy(), np.linalg.svd(c[0],compute_uv=False))
    print(u.cpu().numpy()[0]); print(vt.cpu().numpy()[0])
