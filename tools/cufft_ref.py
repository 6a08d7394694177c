"""Reference point for K1b: cuFFT (torch.fft) doing the same 2D circulant
embedding pass at config 5 (not used by the framework; timing only)."""
import torch

n, M = 1024, 2048
dev = torch.device("cuda")
x = torch.randn(n, n, dtype=torch.complex128, device=dev)
sym = torch.randn(M, M, dtype=torch.float64, device=dev)


def ours_like():
    a = torch.fft.fft(x, n=M, dim=1)              # n rows, padded to M
    b = torch.fft.fft(a, n=M, dim=0)              # M columns, padded
    b *= sym
    c = torch.fft.ifft(b, dim=0)[:n]
    return torch.fft.ifft(c, dim=1)[:, :n]


def full2d():
    xp = torch.zeros(M, M, dtype=torch.complex128, device=dev)
    xp[:n, :n] = x
    return torch.fft.ifft2(torch.fft.fft2(xp) * sym)[:n, :n]


for name, fn in (("row/col pruned", ours_like), ("full 2D", full2d)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"cuFFT {name}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us per 2-RHS pass")
# pure batched line FFTs (no copies): 1024 x 2048 complex128 along dim 1
a = torch.randn(n, M, dtype=torch.complex128, device=dev)
for _ in range(3):
    torch.fft.fft(a, dim=1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    torch.fft.fft(a, dim=1)
e1.record()
torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 50 * 1e3
print(f"cuFFT 1024 lines x 2048 (contiguous): {t:.1f} us = {t / 1024 * 1e3:.1f} ns per line")
