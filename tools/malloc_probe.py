"""cudaMalloc / cudaFree latency on the box (the variance behind model
construction and first-call times): six alloc/free pairs per size, ms."""
import ctypes as C, time, glob, torch
torch.cuda.init(); torch.zeros(1, device="cuda")
libs = glob.glob("/usr/local/cuda/lib64/libcudart.so*") + glob.glob("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/cuda_runtime/lib/libcudart.so*")
rt = C.CDLL(libs[0])
p = C.c_void_p()
for size in (1 << 20, 64 << 20, 1 << 30, 4 << 30):
    ts = []
    for i in range(6):
        t0 = time.perf_counter(); rt.cudaMalloc(C.byref(p), C.c_size_t(size)); t1 = time.perf_counter()
        rt.cudaFree(p); t2 = time.perf_counter()
        ts.append((1e3 * (t1 - t0), 1e3 * (t2 - t1)))
    print(size >> 20, "MiB:", " ".join(f"{a:.2f}/{b:.2f}" for a, b in ts))
