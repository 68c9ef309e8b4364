import ctypes, torch
torch.cuda.init()
rt = ctypes.CDLL("libcudart.so") if False else None
import glob
cands = glob.glob("/usr/local/cuda/lib64/libcudart.so*") + glob.glob("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cuda_runtime/lib/libcudart.so*")
rt = ctypes.CDLL(cands[0])
v = ctypes.c_int()
for name, attr in [("MaxPersistingL2CacheSize", 108), ("MaxAccessPolicyWindowSize", 109), ("L2CacheSize", 89)]:
    rt.cudaDeviceGetAttribute(ctypes.byref(v), attr, 0); print(name, v.value / 2**20, "MiB")
