"""Can cuTensorMapEncodeTiled describe [B, N, H, d] (non-monotonic strides) tensors?  Prints the CUresult per layout."""
import ctypes

import torch

torch.zeros(1, device="cuda")  # a current context for the driver call
cu = ctypes.CDLL("libcuda.so.1")
print("cuInit", cu.cuInit(0))
fn = cu.cuTensorMapEncodeTiled
tm = (ctypes.c_uint8 * 128)()
def enc(dims, strides, box):
    r = len(dims)
    D = (ctypes.c_uint64 * r)(*dims); S = (ctypes.c_uint64 * (r-1))(*strides); B = (ctypes.c_uint32 * r)(*box); E = (ctypes.c_uint32 * r)(*([1]*r))
    # dtype bf16 = 9? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 = 9; interleave none 0; swizzle 128B = 3; l2 promo 0; oob fill none 0
    return fn(tm, 9, r, ctypes.c_void_p(0x10000000), D, S, B, E, 0, 3, 0, 0)
N,H,B,d=16384,12,2,64
print("std  ", enc([d,N,H,B],[d*2, N*d*2, H*N*d*2],[64,128,1,1]))
print("bnhd ", enc([d,N,H,B],[H*d*2, d*2, N*H*d*2],[64,128,1,1]))
print("qkv  ", enc([d,N,H,B],[3*H*d*2, d*2, N*3*H*d*2],[64,128,1,1]))
