"""Probe (dev tooling): cuMulticastCreate with integer handle-type bitmasks."""
from cuda.bindings import driver as cu

cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
err, ctx = cu.cuDevicePrimaryCtxRetain(dev)
cu.cuCtxSetCurrent(ctx)
for ht in (0, 1, 8):
    p = cu.CUmulticastObjectProp()
    p.numDevices = 1
    p.handleTypes = ht
    p.size = 2 << 20
    p.flags = 0
    e2, mc = cu.cuMulticastCreate(p)
    print("handleTypes", ht, "create", e2, p.numDevices, p.handleTypes, p.size)
