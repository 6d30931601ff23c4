"""Cost of pinning a caller's pageable buffer in place (cudaHostRegister /
cudaHostUnregister) against copying it into pinned staging, and the H2D rate
from the registered buffer: decides the host-buffer pipeline design."""
import ctypes, time, torch
cr = torch.cuda.cudart()
dev = torch.device("cuda:0")
torch.cuda.init()
for mb in (8, 64, 256):
    n = mb << 20
    buf = ctypes.create_string_buffer(n)  # pageable, touched
    ctypes.memset(buf, 1, n)
    ptr = ctypes.addressof(buf)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = cr.cudaHostRegister(ptr, n, 0)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record()
        cr.cudaMemcpyAsync(d.data_ptr(), ptr, n, 1, torch.cuda.current_stream().cuda_stream) if hasattr(cr, "cudaMemcpyAsync") else None
        e.record(); torch.cuda.synchronize()
        t2 = time.perf_counter()
        cr.cudaHostUnregister(ptr)
        t3 = time.perf_counter()
        ts.append((int(r), (t1 - t0) * 1e3, (t3 - t2) * 1e3, s.elapsed_time(e)))
    print(mb, "MB register/unregister/copy ms:", ts, flush=True)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    t0 = time.perf_counter(); ctypes.memmove(h.data_ptr(), ptr, n); t1 = time.perf_counter()
    print(mb, "MB single-thread memcpy into pinned ms:", round((t1 - t0) * 1e3, 3), flush=True)
