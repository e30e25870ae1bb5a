"""Probe cuMulticastCreate parameter combinations on this box (ctypes on libcuda)."""
import ctypes
cu = ctypes.CDLL("libcuda.so.1")
print("init", cu.cuInit(0))
dev = ctypes.c_int(); cu.cuDeviceGet(ctypes.byref(dev), 0)
ctx = ctypes.c_void_p(); print("ctx", cu.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), dev), cu.cuCtxSetCurrent(ctx))
class Prop(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong), ("flags", ctypes.c_ulonglong)]
for nd in (1, 2):
    for ht in (0, 1, 8):
        p = Prop(nd, 1 << 21, ht, 0)
        g = ctypes.c_size_t(0)
        r1 = cu.cuMulticastGetGranularity(ctypes.byref(g), ctypes.byref(p), 1)
        p.size = max(1 << 21, g.value)
        h = ctypes.c_ulonglong(0)
        r2 = cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(p))
        r3 = cu.cuMulticastAddDevice(h, dev) if r2 == 0 else -1
        print(f"numDevices={nd} handleTypes={ht}: gran rc={r1} g={g.value} create rc={r2} add rc={r3}")
        if r2 == 0: cu.cuMemRelease(h)
import os
print("imex channels:", os.path.exists("/dev/nvidia-caps-imex-channels"), [l for l in open("/proc/devices") if "imex" in l])
