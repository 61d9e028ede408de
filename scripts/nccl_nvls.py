import torch, torch.distributed as dist
dist.init_process_group("nccl")
r = dist.get_rank(); torch.cuda.set_device(r)
x = torch.ones(1 << 26, dtype=torch.float16, device="cuda")
for _ in range(5): dist.all_reduce(x)
torch.cuda.synchronize()
dist.destroy_process_group()
