"""Probe cuFile on the GPU box: driver open, handle register, one read into device memory
(ctypes, no library code), then the library's SLLM_MODE_GDS on the toy checkpoint.
Every step prints as it completes (run under `timeout`)."""
import ctypes as C
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def say(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


class Descr(C.Structure):
    _fields_ = [("type", C.c_int), ("fd", C.c_int64), ("fs_ops", C.c_void_p)]


class Err(C.Structure):
    _fields_ = [("err", C.c_int), ("cu_err", C.c_int)]


where = sys.argv[1] if len(sys.argv) > 1 else tempfile.gettempdir()
mode = sys.argv[2] if len(sys.argv) > 2 else "raw"
torch.cuda.init()
buf = torch.zeros(8 << 20, dtype=torch.uint8, device="cuda")
say("cuda ready", torch.cuda.get_device_name(0), "dir", where, os.statvfs(where).f_bsize)
path = os.path.join(where, "gds_probe.bin")
data = np.random.default_rng(0).integers(0, 256, 8 << 20, dtype=np.uint8)
data.tofile(path)
if mode == "raw":
    lib = C.CDLL("libcufile.so.0")
    lib.cuFileDriverOpen.restype = Err
    lib.cuFileHandleRegister.restype = Err
    lib.cuFileRead.restype = C.c_ssize_t
    lib.cuFileRead.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int64, C.c_int64]
    e = lib.cuFileDriverOpen()
    say("driver open", e.err, e.cu_err)
    for flags, name in ((os.O_RDONLY | os.O_DIRECT, "O_DIRECT"), (os.O_RDONLY, "buffered")):
        try:
            fd = os.open(path, flags)
        except OSError as ex:
            say(name, "open failed", ex)
            continue
        d = Descr(1, fd, None)
        fh = C.c_void_p()
        e = lib.cuFileHandleRegister(C.byref(fh), C.byref(d))
        say(name, "register", e.err, e.cu_err)
        if e.err == 0:
            t0 = time.perf_counter()
            r = lib.cuFileRead(fh, C.c_void_p(buf.data_ptr()), 8 << 20, 0, 0)
            say(name, "read ->", r, f"{time.perf_counter() - t0:.4f}s",
                "equal" if np.array_equal(buf.cpu().numpy(), data) else "MISMATCH")
            buf.zero_()
            lib.cuFileHandleDeregister(fh)
        os.close(fd)
else:
    import paper_2401_14351_b200 as sllm
    from synth import models, payload
    inv, seed = models.model_inventory("toy")
    payloads = [payload.payload_bytes(seed, e, t.nbytes) for e, t in enumerate(inv)]
    ck = os.path.join(where, "gds_toy")
    os.makedirs(ck, exist_ok=True)
    sllm.convert([(t.name, t.device, t.dtype, t.shape, p.ctypes.data) for t, p in zip(inv, payloads)], ck, 4096,
                 1 << 20, "toy")
    idx = sllm.Index.open(os.path.join(ck, "index.bin"))
    say("converted; loading with mode gds")
    res = sllm.load_files(idx, ck, {0: 0}, sllm.LoadConfig(chunk_bytes=1 << 20, mode="gds"), io_threads=1,
                          stream_of_caller=False)
    say("loaded", res.report)
