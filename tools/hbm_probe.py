"""HBM bandwidth by read/write mix (torch kernels, CUDA events), for the roofline of the
write-heavy sum pass (16 reads : 45 writes) and the read-heavy stream pass (65 : 16)."""
import torch

N = 1 << 29  # 4 GiB of fp64
x = torch.empty(N, dtype=torch.float64, device="cuda")
y = torch.empty(N, dtype=torch.float64, device="cuda")
x.uniform_()


def t(fn, nbytes, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    return nbytes / ms / 1e6


print("write-only (fill_)  GB/s: %.0f" % t(lambda: y.fill_(1.0), 8 * N))
print("read-only  (sum)    GB/s: %.0f" % t(lambda: x.sum(), 8 * N))
print("copy 1:1   (copy_)  GB/s: %.0f" % t(lambda: y.copy_(x), 16 * N))
# 1 read : 3 writes
q = N // 4
xs = x[:q]
ys = [y[i * q:(i + 1) * q] for i in range(3)]
print("1R:3W (3 copies of one source) GB/s: %.0f" %
      t(lambda: [yy.copy_(xs) for yy in ys], 8 * q * 6))
