import sys, ctypes, torch
sys.path.insert(0, '.')
from paper_1505_04650_b200 import _lib
lib = _lib.load()
lib.cnmf_debug_tc.argtypes = [ctypes.c_int, ctypes.c_void_p]
t = int(sys.argv[1])
out = torch.full((256,), -7.0, device="cuda")
st = lib.cnmf_debug_tc(t, out.data_ptr())
print("test", t, "status", st, flush=True)
o = out.cpu().numpy()
print("test", t, o[:8], o[60:68], o[250:256], flush=True)
