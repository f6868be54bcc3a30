import sys, ctypes
sys.path[:0] = ['.', 'tests', 'oracle']
import torch
from test_gpu_compensator import _linear_pe_case
import paper_2605_20659_b200 as P
x, params, pe, grid, W, lin = _linear_pe_case(1, 2, 128, (2, 8, 16), seed=3)
st = P.ForwardSettings(P.SparseSettings(64, topk=1), compensator="linear")
try:
    P.compensator_branch(x, grid, params, st, pe, lin_proj=lin, lin_weights=W)
except Exception as e:
    print("EXC", e)
cudart = ctypes.CDLL("libcudart.so")
cudart.cudaGetErrorString.restype = ctypes.c_char_p
err = cudart.cudaGetLastError()
print("last error", err, cudart.cudaGetErrorString(err))
