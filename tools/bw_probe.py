"""Write-only / read-only / copy HBM bandwidth probe (torch kernels; CUDA events, best of 5)."""
import torch
x = torch.empty(1 << 29, dtype=torch.int64, device="cuda")   # 4 GiB
y = torch.empty(1 << 29, dtype=torch.int64, device="cuda")


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


gb = x.numel() * 8 / 1e9
ms = t(lambda: x.fill_(7))
print(f"fill (write only)   {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s")
ms = t(lambda: x.zero_())
print(f"memset (write only) {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s")
ms = t(lambda: x.sum())
print(f"sum (read only)     {ms:.3f} ms  {gb / ms * 1e3:.0f} GB/s")
ms = t(lambda: y.copy_(x))
print(f"copy (read+write)   {ms:.3f} ms  {2 * gb / ms * 1e3:.0f} GB/s")
