"""Probe (dev tooling): which cuMulticastCreate property combinations this box accepts."""
from cuda.bindings import driver as cu

cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
err, ctx = cu.cuDevicePrimaryCtxRetain(dev)
cu.cuCtxSetCurrent(ctx)
H = cu.CUmemAllocationHandleType
for name, ht in [("NONE", H.CU_MEM_HANDLE_TYPE_NONE), ("FD", H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                 ("FABRIC", H.CU_MEM_HANDLE_TYPE_FABRIC)]:
    for nd in (1, 2):
        p = cu.CUmulticastObjectProp()
        p.numDevices = nd
        p.handleTypes = ht
        p.size = 2 << 20
        e1, g = cu.cuMulticastGetGranularity(p, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        p.size = max(int(g) if e1 == 0 else 0, 2 << 20)
        e2, mc = cu.cuMulticastCreate(p)
        print(name, nd, "gran", e1, g, "create", e2)
        if e2 == 0:
            cu.cuMemRelease(mc)
