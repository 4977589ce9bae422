"""Probe: pitched (2-D) vs 1-D pinned H2D copy bandwidth for one tile (dev tool)."""
import ctypes, glob, os, time
import torch
libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
rt = ctypes.CDLL(sorted(libs)[0])
rt.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_size_t,
                                 ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
rt.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
N, T = 32768, 4096
host = torch.empty((T, N), dtype=torch.float32, pin_memory=True)  # one row band of A (512 MiB)
dev = [torch.empty((T, T), dtype=torch.float32, device="cuda") for _ in range(8)]
streams = [torch.cuda.Stream() for _ in range(8)]
def run(nstreams, two_d=True, reps=2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for r in range(reps):
        for k in range(8):
            s = streams[k % nstreams]
            src = host.data_ptr() + k * T * 4
            if two_d:
                rt.cudaMemcpy2DAsync(dev[k].data_ptr(), T * 4, src, N * 4, T * 4, T, 1, s.cuda_stream)
            else:
                rt.cudaMemcpyAsync(dev[k].data_ptr(), host.data_ptr() + k * T * T * 4, T * T * 4, 1, s.cuda_stream)
    torch.cuda.synchronize()
    return reps * 8 * T * T * 4 / (time.perf_counter() - t0) / 1e9
for ns in (1, 2, 4, 8):
    print(f"2-D tile copies, {ns} streams: {run(ns, True):.1f} GB/s;   1-D 64 MiB copies: {run(ns, False):.1f} GB/s", flush=True)
