"""Driver for ipc_flag_probe.cu: R processes on cuda:0 pass data around a ring through CUDA IPC
memory, signalled by a device-side flag (release atomic / acquire spin), with NO host sync inside
the loop (epoch e uses slot e of the receive buffer).  Checks the data and prints the time per
ring step.   python ipc_flag_probe.py [R] [epochs]"""
import ctypes, os, sys, time
import torch, torch.distributed as dist, torch.multiprocessing as mp

SO = os.environ.get("IPCP_SO", "/tmp/ipcp.so")


def run(rank, R, E):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
    dist.init_process_group("gloo", rank=rank, world_size=R)
    torch.cuda.set_device(0)
    lib = ctypes.CDLL(SO)
    rt = ctypes.CDLL("libcudart.so")
    P = ctypes.c_void_p
    n = 4096
    buf, flag, out, tmo = P(), P(), P(), P()
    for p, b in ((buf, 4 * n * (E + 1)), (flag, 8), (out, 4 * n), (tmo, 4)):
        assert lib.p_malloc(ctypes.c_size_t(b), ctypes.byref(p)) == 0
    h, hf = (ctypes.c_ubyte * 64)(), (ctypes.c_ubyte * 64)()
    assert lib.p_ipc_handle(buf, h) == 0 and lib.p_ipc_handle(flag, hf) == 0
    allh = [None] * R
    dist.all_gather_object(allh, (bytes(h), bytes(hf)))
    nxt, prv = (rank + 1) % R, (rank - 1) % R
    pb, pf = P(), P()
    if nxt == rank:
        pb, pf = buf, flag
    else:
        assert lib.p_ipc_open((ctypes.c_ubyte * 64)(*allh[nxt][0]), ctypes.byref(pb)) == 0
        assert lib.p_ipc_open((ctypes.c_ubyte * 64)(*allh[nxt][1]), ctypes.byref(pf)) == 0
    src = torch.arange(n, dtype=torch.int32, device="cuda") * (rank + 1)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for e in range(1, E + 1):
        slot_peer = ctypes.c_void_p(pb.value + 4 * n * e)
        slot_mine = ctypes.c_void_p(buf.value + 4 * n * e)
        assert lib.p_put(ctypes.c_void_p(src.data_ptr()), slot_peer, n, pf, ctypes.c_ulonglong(e), s) == 0
        assert lib.p_wait(slot_mine, n, flag, ctypes.c_ulonglong(4 * e), out, tmo, s) == 0
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    ob, tb = (ctypes.c_int32 * n)(), (ctypes.c_int32 * 1)()
    rt.cudaMemcpy(ob, out, ctypes.c_size_t(4 * n), 2)
    rt.cudaMemcpy(tb, tmo, ctypes.c_size_t(4), 2)
    exp = [i * (prv + 1) + E for i in range(n)]
    ok = list(ob) == exp and tb[0] == 0
    print(f"rank {rank}/{R}: ok={ok} timeout={tb[0]} {el / E * 1e6:.1f} us per epoch (no host sync)", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    E = int(sys.argv[2]) if len(sys.argv) > 2 else 200
    mp.spawn(run, args=(R, E), nprocs=R)
