import time, numpy as np, torch
x = np.random.default_rng(0).standard_normal(2 * 65536 * 4096).astype(np.float32)
t = torch.from_numpy(x); cr = torch.cuda.cudart(); torch.cuda.init()
for _ in range(2):
    t0 = time.perf_counter(); r = cr.cudaHostRegister(t.data_ptr(), x.nbytes, 0); t1 = time.perf_counter()
    cr.cudaHostUnregister(t.data_ptr()); t2 = time.perf_counter()
    print("register", r, (t1 - t0) * 1e3, "unregister", (t2 - t1) * 1e3)
for _ in range(3):
    t0 = time.perf_counter(); o = torch.empty(x.size, dtype=torch.float32, pin_memory=True); t1 = time.perf_counter()
    print("pinned empty 2GB", (t1 - t0) * 1e3); del o
d = torch.empty(x.size, dtype=torch.float32, device="cuda")
o = torch.empty(x.size, dtype=torch.float32, pin_memory=True)
for _ in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter(); o.copy_(d, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    print("D2H 2GB pinned", (t1 - t0) * 1e3)
