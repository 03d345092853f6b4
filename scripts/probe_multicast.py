"""Probe: can this box create an NVLink multicast object (NVLS, multimem.*)?
Prints the device attributes, then tries cuMulticastCreate with several handle
types / sizes for one device and, on success, AddDevice / BindMem / Map, and
reports each step's CUresult (NEXT-4b feasibility on a one-GPU lease)."""
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
A = D.CUdevice_attribute
for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED"):
    if hasattr(A, name):
        e, v = chk(D.cuDeviceGetAttribute(getattr(A, name), dev))
        out[name.replace("CU_DEVICE_ATTRIBUTE_", "").lower()] = (e, v[0] if v else None)
H = D.CUmemAllocationHandleType
tries = []
for hname in ("CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC"):
    if not hasattr(H, hname):
        continue
    for size in (2 << 20, 512 << 20):
        t = {"handle": hname, "size": size}
        try:
            prop = D.CUmulticastObjectProp()
            prop.numDevices = 1
            prop.size = size
            prop.handleTypes = getattr(H, hname)
            prop.flags = 0
            e, g = chk(D.cuMulticastGetGranularity(prop, D.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM))
            t["granularity"] = (e, int(g[0]) if g else None)
            e, h = chk(D.cuMulticastCreate(prop))
            t["create"] = e
            if e == 0:
                mc = h[0]
                t["add_device"] = chk(D.cuMulticastAddDevice(mc, dev))[0]
                ap = D.CUmemAllocationProp()
                ap.type = D.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
                ap.location.type = D.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
                ap.location.id = 0
                ap.requestedHandleTypes = getattr(H, hname)
                e, mh = chk(D.cuMemCreate(size, ap, 0))
                t["mem_create"] = e
                if e == 0:
                    t["bind"] = chk(D.cuMulticastBindMem(mc, 0, mh[0], 0, size, 0))[0]
                    e, va = chk(D.cuMemAddressReserve(size, 0, 0, 0))
                    t["reserve"] = e
                    if e == 0:
                        t["map"] = chk(D.cuMemMap(va[0], size, 0, mc, 0))[0]
        except Exception as ex:  # noqa: BLE001
            t["exception"] = repr(ex)
        tries.append(t)
out["tries"] = tries
print(json.dumps(out))
