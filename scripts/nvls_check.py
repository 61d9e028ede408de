# Does this box expose NVLink SHARP multicast (NVLS)? Device attribute + NCCL's own log.
import ctypes
import torch
cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuInit(0)
for d in range(torch.cuda.device_count()):
    v = ctypes.c_int()
    # CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
    rc = cuda.cuDeviceGetAttribute(ctypes.byref(v), 132, d)
    print("device", d, "multicast_supported", v.value, "rc", rc)
