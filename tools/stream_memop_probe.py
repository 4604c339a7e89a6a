import torch
from cuda.bindings import driver as d
torch.cuda.init()
x = torch.zeros(16, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
dev = d.cuDeviceGet(0)[1]
for a in ["CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1", "CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS", "CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR"]:
    print(a, d.cuDeviceGetAttribute(getattr(d.CUdevice_attribute, a), dev))
st = d.CUstream(s.cuda_stream)
ptr = d.CUdeviceptr(x.data_ptr())
print("write", d.cuStreamWriteValue32(st, ptr, 5, 0))
print("wait", d.cuStreamWaitValue32(st, ptr, 3, 0))
print("wait+flush", d.cuStreamWaitValue32(st, ptr, 3, 1 << 30))
torch.cuda.synchronize(); print(x[:2])
