"""Probe: does cuTensorMapEncodeTiled accept a stage dimension with a 16-byte stride placed
outermost (box smem layout [stage][col][row][16 B])?"""
import torch
import cuda.bindings.driver as d

torch.cuda.init()
x = torch.zeros(256 * 256 * 201 * 2, dtype=torch.float64, device="cuda")
K, N, T1 = 256, 256, 201
for dims, strides, box, name in [
    ([2, K, N, T1], [T1 * 16, K * T1 * 16, 16], [2, 36, 12, 4], "4d stage-outer"),
    ([2 * T1, K, N], [T1 * 16, K * T1 * 16], [8, 36, 12], "3d stage-inner"),
]:
    r = d.cuTensorMapEncodeTiled(d.CUtensorMapDataType.CU_TENSOR_MAP_DATA_TYPE_FLOAT64, d.cuuint32_t(len(dims)),
                                 x.data_ptr(), [d.cuuint64_t(v) for v in dims], [d.cuuint64_t(v) for v in strides],
                                 [d.cuuint32_t(v) for v in box], [d.cuuint32_t(1)] * len(dims),
                                 d.CUtensorMapInterleave.CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 d.CUtensorMapSwizzle.CU_TENSOR_MAP_SWIZZLE_NONE,
                                 d.CUtensorMapL2promotion.CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 d.CUtensorMapFloatOOBfill.CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
    print(name, r[0])
