"""Probe NVLink SHARP / switch multicast support on this box (NVLS
fan-out): device attributes, and whether a 1-device multicast object can be created,
backed and mapped.  Prints one JSON line."""
import ctypes as C
import json


def main():
    cu = C.CDLL("libcuda.so.1")
    out = {}

    def call(name, *args):
        r = getattr(cu, name)(*args)
        return int(r)

    out["cuInit"] = call("cuInit", 0)
    dev = C.c_int()
    out["cuDeviceGet"] = call("cuDeviceGet", C.byref(dev), 0)
    for name, attr in (("multicast_supported", 132), ("fabric_handle_supported", 128),
                       ("vmm_supported", 102), ("ipc_event_supported", 125)):
        v = C.c_int(-1)
        r = call("cuDeviceGetAttribute", C.byref(v), attr, dev)
        out[name] = v.value if r == 0 else f"err {r}"
    ctx = C.c_void_p()
    out["cuDevicePrimaryCtxRetain"] = call("cuDevicePrimaryCtxRetain", C.byref(ctx), dev)
    call("cuCtxSetCurrent", ctx)

    class MCProp(C.Structure):
        _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t), ("handleTypes", C.c_ulonglong),
                    ("flags", C.c_ulonglong)]

    prop = MCProp(1, 2 << 20, 0, 0)
    gran = C.c_size_t(0)
    out["cuMulticastGetGranularity"] = call("cuMulticastGetGranularity", C.byref(gran), C.byref(prop), 0)
    out["mc_granularity"] = gran.value
    if gran.value:
        prop.size = max(gran.value, 2 << 20)
    h = C.c_ulonglong(0)
    out["cuMulticastCreate"] = call("cuMulticastCreate", C.byref(h), C.byref(prop))
    if out["cuMulticastCreate"] == 0:
        out["cuMulticastAddDevice"] = call("cuMulticastAddDevice", h, dev)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
