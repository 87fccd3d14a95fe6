import os, sys, time
t0 = time.time()
import torch
torch.cuda.init(); torch.zeros(1, device="cuda")
t1 = time.time()
sys.path.insert(0, os.getcwd())
import paper_1612_01506_b200 as sm
lib = sm.load_library()
t2 = time.time()
t = torch.randint(0, 4, (1 << 20,), dtype=torch.uint8, device="cuda")
for m in (4, 300):
    p = bytes(t[1000:1000 + m].cpu().numpy())
    a = time.time(); c = sm.sm_count(p, t); torch.cuda.synchronize(); b = time.time()
    print(f"{os.environ.get('SMGPU_LIB','release')}: first sm_count m={m}: {b - a:.2f} s", flush=True)
print(f"{os.environ.get('SMGPU_LIB','release')}: torch init {t1 - t0:.1f} s, load_library {t2 - t1:.2f} s", flush=True)
