"""Which multicast-object properties does cuMulticastCreate accept on this box?"""
import ctypes

cuda = ctypes.CDLL("libcuda.so.1")
print("init", cuda.cuInit(0))
dev = ctypes.c_int()
cuda.cuDeviceGet(ctypes.byref(dev), 0)
ctx = ctypes.c_void_p()
print("retain", cuda.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev), cuda.cuCtxSetCurrent(ctx))


class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t),
                ("handleTypes", ctypes.c_ulonglong), ("flags", ctypes.c_ulonglong)]


for ht, name in ((0x8, "FABRIC"), (0x1, "POSIX_FD"), (0x0, "NONE")):
    for nd in (1, 2):
        p = Prop(nd, 1 << 21, ht, 0)
        g = ctypes.c_size_t()
        rg = cuda.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(p), 1)
        p.size = max(g.value, 1 << 21) if rg == 0 else (1 << 21)
        h = ctypes.c_ulonglong()
        r = cuda.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
        extra = ""
        if r == 0:
            ra = cuda.cuMulticastAddDevice(h, dev)
            extra = f" add={ra}"
            if ht == 0x8:
                buf = ctypes.create_string_buffer(64)
                extra += f" export={cuda.cuMemExportToShareableHandle(buf, h, 0x8, ctypes.c_ulonglong(0))}"
            cuda.cuMemRelease(h)
        print(f"{name} numDevices={nd}: gran rc={rg} g={g.value} create={r}{extra}")
