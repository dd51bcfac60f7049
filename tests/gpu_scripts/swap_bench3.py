"""Swap bandwidth, P2P kernel vs NCCL (env QSV_SWAP_MODE), via the qsv_swap C-ABI."""
import os, sys, time, ctypes as C
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch, torch.distributed as dist
import paper_2509_04955_b200 as pkg
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
obj = [pkg.Engine.comm_unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
L = pkg.load_qsv()
ctx = C.c_void_p()
assert L.qsv_ctx_create(local, rank, world, C.create_string_buffer(obj[0], 128), C.byref(ctx)) == 0
l = int(sys.argv[1]) if len(sys.argv) > 1 else 29
st = C.c_void_p(); nb = C.c_size_t()
assert L.qsv_state_alloc(ctx, l, C.byref(st), C.byref(nb)) == 0
L.qsv_state_set_basis(st, C.c_uint64(0))
for v in (l - 1, 12, 5):
    cl = min(26, l - 3)
    L.qsv_swap(st, l, v, cl, 2); L.qsv_sync(ctx); dist.barrier()
    t = time.perf_counter()
    reps = 4
    for _ in range(reps):
        rc = L.qsv_swap(st, l, v, cl, 2)
        assert rc == 0, L.qsv_last_error()
    L.qsv_sync(ctx); dist.barrier()
    dt = (time.perf_counter() - t) / reps
    if rank == 0:
        print(f"mode={os.environ.get('QSV_SWAP_MODE', 'p2p')} N={world} l={l} v={v}: {dt*1e3:.2f} ms/swap, "
              f"{16*2**(l-1)/dt/1e9:.0f} GB/s per direction", flush=True)
dist.destroy_process_group()
