import ctypes, torch, numpy as np
cudart = ctypes.CDLL("libcudart.so.12") if False else None
t = torch.empty(1 << 20, dtype=torch.uint8, pin_memory=True)
print("is_pinned (torch):", t.is_pinned())
from cuda.bindings import runtime as rt
err, attr = rt.cudaPointerGetAttributes(t.data_ptr())
print(err, attr.type if hasattr(attr, "type") else attr)
a = np.zeros(1 << 20, np.uint8)
err, attr = rt.cudaPointerGetAttributes(a.ctypes.data)
print(err, attr.type if hasattr(attr, "type") else attr)
