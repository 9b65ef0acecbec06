"""Probe: can two NCCL ranks share one GPU (the gpurun box has one)?  Run under
torchrun --nproc-per-node 2; prints per-rank outcome of a send/recv pair."""
import os
import torch
import torch.distributed as dist

rank = int(os.environ["RANK"])
torch.cuda.set_device(0)
try:
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    t = torch.full((1 << 20,), float(rank), device="cuda")
    r = torch.empty_like(t)
    ops = [dist.P2POp(dist.isend, t, 1 - rank), dist.P2POp(dist.irecv, r, 1 - rank)]
    for q in dist.batch_isend_irecv(ops):
        q.wait()
    torch.cuda.synchronize()
    print(f"rank {rank}: nccl p2p on a shared GPU OK, got {r[0].item()}", flush=True)
    dist.destroy_process_group()
except Exception as e:  # noqa: BLE001
    print(f"rank {rank}: nccl on a shared GPU FAILED: {str(e).splitlines()[0][:300]}", flush=True)
