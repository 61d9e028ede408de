# NVLS probe (torchrun, N GPUs): multicast support, correctness of a switch-reduced fp16
# allreduce vs the exact fp32 sum, and its time/bus bandwidth vs NCCL on the same bytes.
import ctypes, os, sys, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl")
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "nvls_probe.so"))
cu = ctypes.CDLL("libcuda.so.1"); cu.cuInit(0)
v = ctypes.c_int()
cu.cuDeviceGetAttribute(ctypes.byref(v), 132, rank)  # CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED
print(f"rank {rank} multicast_supported {v.value}", flush=True)
sizes = [int(x) for x in os.environ.get("NVLS_BYTES", "51114064,122201680").split(",")]
NBYTES = max(sizes)
buf = symm.empty(NBYTES // 2 + 64, dtype=torch.float16, device="cuda")
h = symm.rendezvous(buf, dist.group.WORLD)
flag = symm.empty(148 * 32, dtype=torch.int32, device="cuda"); flag.zero_()
hf = symm.rendezvous(flag, dist.group.WORLD)
dist.barrier(); torch.cuda.synchronize()
mc = h.multicast_ptr
print(f"rank {rank} multicast_ptr {mc:#x}", flush=True)
if not mc:
    sys.exit(0)
fl = (ctypes.c_void_p * world)(*hf.buffer_ptrs)
epoch = [0]
blocks = int(os.environ.get("NVLS_BLOCKS", "148"))
def run(nbytes, acc32):
    epoch[0] += 1
    rc = lib.nvls_run(ctypes.c_void_p(mc), ctypes.c_size_t(nbytes), rank, world, fl,
                      ctypes.c_uint32(epoch[0]), blocks, acc32,
                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0, rc
for nbytes in sizes:
    n = nbytes // 2
    g = torch.Generator(device="cuda"); g.manual_seed(1234 + rank)
    x = (torch.rand(n, generator=g, device="cuda") * 2 - 1)
    buf[:n].copy_(x.half())
    allx = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(allx, buf[:n].float())
    exact = sum(allx)  # fp32 sum of the fp16 inputs
    torch.cuda.synchronize(); dist.barrier()
    run(nbytes, 1); torch.cuda.synchronize()
    got = buf[:n].float()
    err = ((got - exact).abs() / exact.abs().clamp(min=1)).max().item()
    same = torch.equal(got, exact.half().float())
    ref = buf[:n].clone()
    res = {}
    for acc in (1, 0):
        for _ in range(3): run(nbytes, acc)
        torch.cuda.synchronize(); dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        K = 20
        e0.record()
        for _ in range(K): run(nbytes, acc)
        e1.record(); torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / K], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[acc] = t.item()
    y = torch.empty(n, dtype=torch.float16, device="cuda")
    for _ in range(3): dist.all_reduce(y)
    torch.cuda.synchronize(); dist.barrier()
    e0.record()
    for _ in range(20): dist.all_reduce(y)
    e1.record(); torch.cuda.synchronize()
    tn = torch.tensor([e0.elapsed_time(e1) / 20], device="cuda")
    dist.all_reduce(tn, op=dist.ReduceOp.MAX)
    if rank == 0:
        bus = lambda ms: 2 * (world - 1) / world * nbytes / (ms * 1e-3) / 1e9
        print(f"NVLS N={world} bytes={nbytes} acc32: {res[1]*1e3:.1f} us ({bus(res[1]):.0f} GB/s bus) "
              f"acc16: {res[0]*1e3:.1f} us  nccl: {tn.item()*1e3:.1f} us ({bus(tn.item()):.0f}) "
              f"max_rel_err(acc32 vs exact)={err:.2e} equals_round(exact)={same} blocks={blocks}",
              flush=True)
dist.barrier()
dist.destroy_process_group()
