"""Worker of test_gpu_pregen.test_pregen_two_processes_ipc (torchrun, 2 ranks, 2 GPUs): rank 0
owns the synchronizer, rank 1 maps it over NVLink (CUDA IPC) and arrives on it."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08862_b200 as bs  # noqa: E402

rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
obj = [None]
if rank == 0:
    sync = bs.BubbleSync(0)
    obj = [sync.export()]
dist.broadcast_object_list(obj, src=0)
if rank == 1:
    sync = bs.BubbleSync(1, handle=obj[0])
    sync.arrive(1, 5)
    torch.cuda.synchronize()
dist.barrier()
halt = torch.zeros(1, dtype=torch.int32, device="cuda")
sync.poll(2, 5, halt)
torch.cuda.synchronize()
first = int(halt.item())
if rank == 0:
    sync.arrive(0, 5)
    torch.cuda.synchronize()
dist.barrier()
sync.poll(2, 5, halt)
torch.cuda.synchronize()
assert first == 0 and int(halt.item()) == 1, (rank, first, int(halt.item()))
dist.barrier()
sync.close()
if rank == 0:
    print("ipc poll ok", flush=True)
dist.destroy_process_group()
