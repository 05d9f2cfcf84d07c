"""Write-only / read-only / copy HBM bandwidth on this B200 (torch kernels + cudaMemset), to
put the write-dominated GRID kernel's fraction in context."""
import torch

x = torch.empty(11 * 2**30 // 4, dtype=torch.float32, device="cuda")
y = torch.empty_like(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t(fn, nbytes, name, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name:28s} {nbytes / ms / 1e6:8.0f} GB/s")


n = x.numel() * 4
t(lambda: x.zero_(), n, "write (zero_ / memset)")
t(lambda: x.fill_(0.5), n, "write (fill_ 0.5)")
t(lambda: x.sum(), n, "read (sum)")
t(lambda: y.copy_(x), 2 * n, "copy (read + write)")
