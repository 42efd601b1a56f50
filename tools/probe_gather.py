"""Probe (dev tooling): does gloo all_gather_into_tensor accept CUDA tensors (2 ranks, 1 GPU)?"""
import os
import torch
import torch.distributed as dist

dist.init_process_group("gloo")
r = dist.get_rank()
x = torch.full((4,), float(r), device="cuda:0")
out = torch.empty(8, device="cuda:0")
try:
    dist.all_gather_into_tensor(out, x)
    print(r, "ok", out.tolist())
except Exception as e:  # noqa: BLE001
    print(r, "fail", repr(e)[:200])
dist.destroy_process_group()
