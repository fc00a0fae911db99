"""Host<->device link probe and e2e pipeline sweep (run on the GPU box)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

def bw(n_bytes=2 << 30):
    h = torch.empty(n_bytes // 8, dtype=torch.float64, pin_memory=True)
    d = torch.empty_like(h, device="cuda")
    h2 = torch.empty_like(h, pin_memory=True)
    for _ in range(2):
        d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); h2d = n_bytes / (time.perf_counter() - t)
    t = time.perf_counter(); h2.copy_(d, non_blocking=True); torch.cuda.synchronize(); d2h = n_bytes / (time.perf_counter() - t)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    t = time.perf_counter()
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    d2 = torch.empty_like(d)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); both = 2 * n_bytes / (time.perf_counter() - t)
    return {"h2d_gbs": h2d / 1e9, "d2h_gbs": d2h / 1e9, "duplex_total_gbs": both / 1e9}

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "e2e":
        import numpy as np
        from paper_1401_6235_b200 import kernels as K
        n = 1 << 27
        x = [torch.rand(n, dtype=torch.float64, pin_memory=True).numpy() for _ in range(4)]
        out = K.empty_twofold(n, np.float64, device="cpu", pin_memory=True)
        X, Y = K.TwofoldArray(x[0], x[1]), K.TwofoldArray(x[2], x[3])
        K.vtadd2(X, Y, out)
        t = time.perf_counter()
        for _ in range(3): K.vtadd2(X, Y, out)
        dt = (time.perf_counter() - t) / 3
        print(json.dumps({"slots": os.environ.get("TF_HOST_SLOTS"), "chunk_mb": os.environ.get("TF_HOST_CHUNK_MB"),
                          "melem_s": n / dt / 1e6, "h2d_gbs": 32 * n / dt / 1e9}))
    else:
        print(json.dumps(bw()))
