import os, sys, threading, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
from paper_1510_06585_b200 import marrow as M, trees
H, W = 333, 515
gray = synth.np_u8_stream(8, 0, H * W).reshape(H, W)
gid = os.urandom(128)
t0 = time.time()
import ctypes
cudart = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
MODE = os.environ.get("XR_STREAM", "torch")
def mkstream():
    if MODE == "torch":
        return torch.cuda.Stream()
    h = ctypes.c_void_p()
    lib = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
    assert lib.cudaStreamCreateWithFlags(ctypes.byref(h), 1) == 0
    return torch.cuda.ExternalStream(h.value)
def worker(r):
    torch.cuda.set_device(0)
    s = mkstream()
    print("rank", r, "stream", hex(s.cuda_stream), flush=True)
    with torch.cuda.stream(s):
        c = M.mw_ctx_create(0, r, 2, 1, gid, transport=M.MW_TRANSPORT_LOOPBACK)
        node = trees.hysteresis()
        off, ln = M.mw_partition(c, node, H)
        s0, s1 = off[r], off[r] + ln[r]
        src = torch.from_numpy(np.ascontiguousarray(gray[s0:s1])).cuda()
        dst = torch.empty_like(src)
        print(f"{time.time()-t0:.3f} rank {r} run", flush=True)
        f = M.mw_run(c, node, [M.arg(src, local_offset=s0, global_shape=(H, W)), M.arg(dst, local_offset=s0, global_shape=(H, W))])
        print(f"{time.time()-t0:.3f} rank {r} enqueued", flush=True)
        try:
            print(r, f.wait().result(), flush=True)
        except Exception as e:
            print(r, "ERR", e, flush=True)
        print(f"{time.time()-t0:.3f} rank {r} done", flush=True)
th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
[t.start() for t in th]; [t.join() for t in th]
