import ctypes as C, numpy as np, torch, sys
lib = C.CDLL("tools/libisvd_dbg.so")
s=3
rng=np.random.default_rng(s)
c=rng.standard_normal((1,s,s)); c[0,-1,:]=0
d=torch.tensor(c,device="cuda"); u=torch.empty_like(d); vt=torch.empty_like(d); sv=torch.empty((1,s),dtype=torch.float64,device="cuda")
rc = lib.isvd_core_svd(1,s,C.c_void_p(d.data_ptr()),C.c_void_p(u.data_ptr()),C.c_void_p(sv.data_ptr()),C.c_void_p(vt.data_ptr()),None)
torch.cuda.synchronize()
print(rc, sv.cpu().numpy())
