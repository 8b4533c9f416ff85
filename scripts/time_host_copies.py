"""Host <-> device copy costs of the numpy drop-in path (41.5 MB map D2H,
13.4 MB inputs H2D) under different host-buffer strategies."""
import os
import statistics
import sys
import time

import numpy as np
import torch

n_out = 80 * 360 * 360
dev_out = torch.randn(n_out, device="cuda")
feats = np.random.rand(6, 80, 32, 88).astype(np.float32)


def t(fn, n=10):
    fn()
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


print(f"threads {torch.get_num_threads()}")
print(f"H2D from_numpy().cuda()       {t(lambda: torch.from_numpy(feats).cuda()):7.2f} ms")
print(f"D2H .cpu()                    {t(lambda: dev_out.cpu()):7.2f} ms")
print(f"np.empty + touch (1 thread)   {t(lambda: np.empty(n_out, np.float32).fill(0)):7.2f} ms")


def prefault_copy():
    h = torch.empty(n_out)
    h.zero_()  # multi-threaded first touch
    h.copy_(dev_out)
    return h.numpy()


print(f"D2H into pre-faulted (zero_)  {t(prefault_copy):7.2f} ms")
pinned = torch.empty(n_out, pin_memory=True)
print(f"D2H into cached pinned        {t(lambda: pinned.copy_(dev_out)):7.2f} ms")


def pinned_then_copy():
    pinned.copy_(dev_out)
    out = torch.empty(n_out)
    out.copy_(pinned)  # multi-threaded host copy
    return out.numpy()


print(f"pinned D2H + host copy        {t(pinned_then_copy):7.2f} ms")
print(f"pin_memory alloc              {t(lambda: torch.empty(n_out, pin_memory=True)):7.2f} ms")
