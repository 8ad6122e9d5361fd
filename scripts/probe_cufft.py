"""Context for the FFT row: torch.fft (cuFFT) fft -> ifft over the same
512 x 65536 complex64 batch, CUDA events, vs bench.py --workload fft."""
import torch
x = torch.randn(512, 65536, dtype=torch.complex64, device="cuda")
for _ in range(5):
    y = torch.fft.ifft(torch.fft.fft(x, dim=1), dim=1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 50
e0.record()
for _ in range(K):
    y = torch.fft.ifft(torch.fft.fft(x, dim=1), dim=1)
e1.record(); torch.cuda.synchronize()
print(f"cuFFT fft->ifft 512x65536 c64: {e0.elapsed_time(e1) / K:.4f} ms per batch")
f = torch.empty_like(x)
e0.record()
for _ in range(K):
    torch.fft.fft(x, dim=1, out=f)
e1.record(); torch.cuda.synchronize()
print(f"cuFFT fft only: {e0.elapsed_time(e1) / K:.4f} ms per batch")
