"""One rank of the host-only protocol test of tests/shim (test_nccl_shim.py): grouped
send/recv allgather of uneven slices and grouped allreduce (sum f64, max i32),
50 rounds, through the shim built with -DHMX_SHIM_HOST_ONLY."""
import ctypes, os, sys, numpy as np
lib = ctypes.CDLL(sys.argv[1]); rank, world = int(sys.argv[2]), int(sys.argv[3]); idfile = sys.argv[4]
class UID(ctypes.Structure): _fields_ = [("internal", ctypes.c_char * 128)]
uid = UID()
if rank == 0:
    lib.ncclGetUniqueId(ctypes.byref(uid)); open(idfile + ".tmp", "wb").write(bytes(uid)); os.replace(idfile + ".tmp", idfile)
else:
    import time
    while not os.path.exists(idfile): time.sleep(0.01)
    ctypes.memmove(ctypes.byref(uid), open(idfile, "rb").read(), 128)
comm = ctypes.c_void_p()
assert lib.ncclCommInitRank(ctypes.byref(comm), world, uid, rank) == 0
n = 1000
cuts = [n * k // world for k in range(world + 1)]
for it in range(50):
    full = np.zeros(n); full[cuts[rank]:cuts[rank+1]] = rank + it
    lib.ncclGroupStart()
    for q in range(world):
        if q == rank: continue
        m = cuts[rank+1] - cuts[rank]; mq = cuts[q+1] - cuts[q]
        assert lib.ncclSend(ctypes.c_void_p(full.ctypes.data + 8*cuts[rank]), ctypes.c_size_t(m), 8, q, comm, None) == 0
        assert lib.ncclRecv(ctypes.c_void_p(full.ctypes.data + 8*cuts[q]), ctypes.c_size_t(mq), 8, q, comm, None) == 0
    assert lib.ncclGroupEnd() == 0
    for q in range(world):
        assert np.all(full[cuts[q]:cuts[q+1]] == q + it), (it, q)
    v = np.array([rank + 1.0, it], dtype=np.float64); fl = np.array([rank], dtype=np.int32)
    lib.ncclGroupStart()
    assert lib.ncclAllReduce(ctypes.c_void_p(v.ctypes.data), ctypes.c_void_p(v.ctypes.data), ctypes.c_size_t(2), 8, 0, comm, None) == 0
    assert lib.ncclAllReduce(ctypes.c_void_p(fl.ctypes.data), ctypes.c_void_p(fl.ctypes.data), ctypes.c_size_t(1), 2, 2, comm, None) == 0
    assert lib.ncclGroupEnd() == 0
    assert v[0] == world * (world + 1) / 2 and v[1] == it * world and fl[0] == world - 1, (v, fl)
assert lib.ncclCommDestroy(comm) == 0
print("rank", rank, "ok")
