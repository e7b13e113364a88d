import ctypes
cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuInit(0)
dev = ctypes.c_int()
cuda.cuDeviceGet(ctypes.byref(dev), 0)
v = ctypes.c_int()
# CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
r = cuda.cuDeviceGetAttribute(ctypes.byref(v), 132, dev)
print("multicast supported attr:", r, v.value)
