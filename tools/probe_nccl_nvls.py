"""Probe: can this box run the fused NVLS merge (NEXT-f3) through NCCL's symmetric windows?

    NCCL_DEBUG=INFO python tools/probe_nccl_nvls.py > profiles/r02_nvls_probe.log 2>&1

Prints the device's multicast attribute (cuda driver API), the NCCL version, then tries the library's
GRCA_MERGE_NVLS binding on a one-rank communicator (ncclMemAlloc + ncclCommWindowRegister +
ncclDevCommCreate(lsaMultimem) + the lsa multimem pointer) and reports the outcome verbatim.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import scenegen as sg  # noqa: E402
from paper_2605_10457_b200 import Grca, GrcaError  # noqa: E402
from paper_2605_10457_b200 import grca as G  # noqa: E402


def main():
    print("torch", torch.__version__, "nccl", torch.cuda.nccl.version(), "devices", torch.cuda.device_count())
    try:
        from cuda.bindings import driver as cu

        cu.cuInit(0)
        _, dev = cu.cuDeviceGet(0)
        _, mc = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
        _, fab = cu.cuDeviceGetAttribute(
            cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev)
        print("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED =", mc, " HANDLE_TYPE_FABRIC_SUPPORTED =", fab)
    except Exception as e:  # noqa: BLE001
        print("driver-API query failed:", e)
    print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
    ems, tris = sg.random_scene(61, n_tris=300, n_emitters=1, gamma=8, chi=64)
    g = Grca(device=0, max_triangles=len(tris), max_rays=sg.n_rays_total(ems), nranks=1, rank=0,
             nccl_uid=G.nccl_unique_id(), shard_mode=G.SHARD_TRIANGLES, merge=G.MERGE_NVLS)
    try:
        g.set_emitters(ems)
        print("GRCA_MERGE_NVLS bound: multimem pointer obtained (fused merge runnable)")
    except GrcaError as e:
        print("GRCA_MERGE_NVLS binding failed:", e)
    g.close()


if __name__ == "__main__":
    main()
