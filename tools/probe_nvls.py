"""Probe (dev tooling): multicast / NVLS availability on this box, via torch symmetric memory and
the CUDA driver attribute.  Prints one JSON line."""
import json
import os

import torch
import torch.distributed as dist

out = {}
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
try:
    from cuda.bindings import driver as cu
    cu.cuInit(0)
    err, dev = cu.cuDeviceGet(0)
    err, mc = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    out["driver_multicast_supported"] = int(mc)
    err, fab = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev)
    out["fabric_handles"] = int(fab)
except Exception as e:  # noqa: BLE001
    out["driver_error"] = repr(e)[:200]
try:
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1024, dtype=torch.int64, device="cuda:0")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    out["symm_multicast_ptr"] = int(getattr(h, "multicast_ptr", 0) or 0)
    out["symm_buffer_ptr0"] = int(h.buffer_ptrs[0]) if hasattr(h, "buffer_ptrs") else None
    out["symm_backend"] = str(getattr(symm, "get_backend", lambda *a: "?")("cuda:0")) if hasattr(symm, "get_backend") else "?"
    dist.destroy_process_group()
except Exception as e:  # noqa: BLE001
    out["symm_error"] = repr(e)[:300]
print(json.dumps(out))
