"""Copy-engine bandwidth into CUDA-IPC memory with explicit cudaMemcpyPeerAsync /
cudaMemcpyAsync (2 processes, 2 GPUs), after cudaDeviceEnablePeerAccess."""
import ctypes
import glob
import os

import torch
import torch.multiprocessing as mp


def rt():
    libs = glob.glob("/usr/local/cuda/lib64/libcudart.so*")
    return ctypes.CDLL(sorted(libs)[0])


def child(q, done):
    torch.cuda.set_device(1)
    torch.zeros(1, device="cuda:1")
    r = rt()
    print("enable peer 1->0:", r.cudaDeviceEnablePeerAccess(0, 0), flush=True)
    peer = q.get()
    src = torch.ones(peer.numel(), dtype=peer.dtype, device="cuda:1")
    s = torch.cuda.Stream(device="cuda:1")
    n = 32 << 20  # bytes
    for kind in ("peer", "async"):
        def go():
            if kind == "peer":
                return r.cudaMemcpyPeerAsync(ctypes.c_void_p(peer.data_ptr()), 0,
                                             ctypes.c_void_p(src.data_ptr()), 1,
                                             ctypes.c_size_t(n), ctypes.c_void_p(s.cuda_stream))
            return r.cudaMemcpyAsync(ctypes.c_void_p(peer.data_ptr()),
                                     ctypes.c_void_p(src.data_ptr()), ctypes.c_size_t(n), 3,
                                     ctypes.c_void_p(s.cuda_stream))
        for _ in range(3):
            rc = go()
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            go()
        e1.record(s)
        s.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"{kind}: rc={rc} {n / ms / 1e6:.1f} GB/s", flush=True)
    done.put(1)


if __name__ == "__main__":
    mp.set_start_method("spawn")
    q, done = mp.Queue(), mp.Queue()
    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda:0")
    print("enable peer 0->1:", rt().cudaDeviceEnablePeerAccess(1, 0), flush=True)
    buf = torch.zeros(64 << 20, dtype=torch.bfloat16, device="cuda:0")
    p = mp.Process(target=child, args=(q, done))
    p.start()
    q.put(buf)
    done.get()
    p.join()
    os._exit(0)
