"""Probe: does this box support CUDA multicast objects (NVLS, multimem.st)?"""
import ctypes
cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = ctypes.c_int()
cu.cuDeviceGet(ctypes.byref(dev), 0)
for name, attr in (("MULTICAST_SUPPORTED", 132), ("HANDLE_TYPE_FABRIC_SUPPORTED", 128), ("IPC_EVENT_SUPPORTED", 125)):
    v = ctypes.c_int(-1)
    r = cu.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
    print(name, "rc", r, "value", v.value)
