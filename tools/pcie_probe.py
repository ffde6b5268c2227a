"""PCIe probe: pinned H2D alone, D2H alone, and both at once (separate streams), in GB/s,
with copy sizes like the e2e path's (1.416 GB scene upload; 33 MB frames)."""
import time
import torch

def bw(fn, nbytes, reps=5):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t) / 1e9

S = 1_416_000_000 // 4
F = 33_177_600 // 4
h_in = torch.empty(S, pin_memory=True)
d_in = torch.empty(S, device="cuda")
d_fr = torch.empty(64, F, device="cuda")
h_fr = torch.empty(64, F, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2):
        for i in range(64):
            h_fr[i].copy_(d_fr[i], non_blocking=True)
def both():
    h2d(); d2h()

print(f"H2D alone {bw(h2d, S * 4):.1f} GB/s")
print(f"D2H alone (64 x 33 MB) {bw(d2h, 64 * F * 4):.1f} GB/s")
t = time.perf_counter()
for _ in range(5):
    both()
torch.cuda.synchronize()
el = time.perf_counter() - t
print(f"both at once: {5 * (S + 64 * F) * 4 / el / 1e9:.1f} GB/s total ({5 * S * 4 / el / 1e9:.1f} + {5 * 64 * F * 4 / el / 1e9:.1f} if both spanned the run)")
