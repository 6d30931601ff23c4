"""What a plain device copy achieves at C1 sizes (rotating 16 buffers,
back-to-back launches, CUDA events): the practical floor the C1 kernels are
compared with. Prints us and GB/s per copy size."""
import torch

dev = torch.device("cuda:0")
R = 16
for label, nbytes_in, nbytes_out in (("copy 32MB->32MB (dequant-sized writes)", 32 << 20, 32 << 20),
                                     ("copy 8MB->8MB", 8 << 20, 8 << 20),
                                     ("copy 42.5MB->42.5MB", 42467328, 42467328)):
    xs = [torch.empty(nbytes_in, dtype=torch.uint8, device=dev).fill_(1) for _ in range(R)]
    ys = [torch.empty(nbytes_out, dtype=torch.uint8, device=dev) for _ in range(R)]
    for i in range(R):
        ys[i].copy_(xs[i])
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    it = 80
    s.record()
    for i in range(it):
        ys[i % R].copy_(xs[i % R])
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) * 1e3 / it
    print(f"{label}: {us:.2f} us, {(nbytes_in + nbytes_out) / us / 1e3:.0f} GB/s", flush=True)
    del xs, ys
