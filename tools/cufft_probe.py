import torch, time
z = torch.randn(32, 256, 256, dtype=torch.complex128, device="cuda")
for f in (torch.fft.fft2, torch.fft.ifft2):
    y = f(z); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, f in (("fft2", torch.fft.fft2), ("ifft2", torch.fft.ifft2)):
    e0.record()
    for _ in range(50):
        y = f(z)
    e1.record(); torch.cuda.synchronize()
    print(name, "32 x 256^2 complex128:", round(e0.elapsed_time(e1) / 50 * 1e3, 1), "us")
# in-place style with preallocated out
out = torch.empty_like(z)
e0.record()
for _ in range(50):
    torch.fft.fft2(z, out=out)
e1.record(); torch.cuda.synchronize()
print("fft2(out=)", round(e0.elapsed_time(e1) / 50 * 1e3, 1), "us")
