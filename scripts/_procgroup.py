"""Process-group set-up shared by the torchrun check scripts.

One process per GPU normally (NCCL host group).  With more processes than
GPUs (e.g. the 8-process placement on a 4-GPU box) the processes share the
GPUs round-robin and the host group is gloo, since NCCL puts at most one rank
on a GPU; the device-side sync (IPC + device signals) is unchanged.
"""

import os

import torch
import torch.distributed as dist


def init() -> int:
    """Initialise the default group; returns this process's CUDA device."""
    local = int(os.environ["LOCAL_RANK"])
    if int(os.environ["WORLD_SIZE"]) > torch.cuda.device_count():
        local %= torch.cuda.device_count()
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return local


def shared() -> bool:
    return dist.get_backend() != "nccl"
