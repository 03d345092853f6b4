"""Probe: can this box create an NVLink multicast object (NVLS, multimem.*)?
Prints the device attribute, then tries cuMulticastCreate / AddDevice / BindMem /
Map for one device and reports each step's result."""
import json
try:
    from cuda.bindings import driver as D
except Exception:  # older cuda-python
    from cuda import cuda as D


def chk(r):
    err = r[0] if isinstance(r, tuple) else r
    return int(err), (r[1:] if isinstance(r, tuple) and len(r) > 1 else None)


out = {}
chk(D.cuInit(0))
e, (dev,) = chk(D.cuDeviceGet(0))
e, (ctx,) = chk(D.cuDevicePrimaryCtxRetain(dev))
chk(D.cuCtxSetCurrent(ctx))
e, v = chk(D.cuDeviceGetAttribute(D.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
out["multicast_supported"] = (e, v[0] if v else None)
try:
    prop = D.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.size = 2 << 20
    prop.handleTypes = D.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
    e, g = chk(D.cuMulticastGetGranularity(prop, D.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
    out["granularity"] = (e, int(g[0]) if g else None)
    e, h = chk(D.cuMulticastCreate(prop))
    out["create"] = e
    if e == 0:
        mc = h[0]
        out["add_device"] = chk(D.cuMulticastAddDevice(mc, dev))[0]
except Exception as ex:  # noqa: BLE001
    out["exception"] = repr(ex)
print(json.dumps(out))
