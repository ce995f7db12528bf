"""Copy-engine bandwidth into a CUDA-IPC-mapped peer buffer (2 processes, 2 GPUs).
Process 1 maps a tensor allocated by process 0 and copies into it with
cudaMemcpyAsync (tensor.copy_), timed with events."""
import time

import torch
import torch.multiprocessing as mp


def child(q, done):
    import ctypes
    import glob
    import os
    torch.cuda.set_device(1)
    torch.zeros(1, device="cuda:1")
    if os.environ.get("ENABLE_PEER"):
        libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart*.so*"))
        libs += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
        rt = ctypes.CDLL(libs[0])
        print("enable peer:", rt.cudaDeviceEnablePeerAccess(0, 0), flush=True)
    peer = q.get()  # mapped into this process via CUDA IPC (lives on GPU 0)
    src = torch.ones(peer.numel(), dtype=peer.dtype, device="cuda:1")
    s = torch.cuda.Stream()
    for mb in (8, 32, 128):
        n = mb * (1 << 20) // 2
        for _ in range(3):
            with torch.cuda.stream(s):
                peer[:n].copy_(src[:n], non_blocking=True)
        s.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(10):
            with torch.cuda.stream(s):
                peer[:n].copy_(src[:n], non_blocking=True)
        e1.record(s)
        s.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(f"IPC CE copy {mb} MB: {ms * 1e3:.1f} us  {n * 2 / ms / 1e6:.1f} GB/s", flush=True)
    done.put(1)


if __name__ == "__main__":
    mp.set_start_method("spawn")
    q, done = mp.Queue(), mp.Queue()
    torch.cuda.set_device(0)
    buf = torch.zeros(64 << 20, dtype=torch.bfloat16, device="cuda:0")
    p = mp.Process(target=child, args=(q, done))
    p.start()
    q.put(buf)
    done.get()
    p.join()
