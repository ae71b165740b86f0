// pwadv_roles.cu — K6: the reference's array-level stencil entry points on
// the GPU:
//
//  * compute_block (pkg/src/pwadvect/kernel.py:139-162): su/sv/sw of columns
//    given the 17 role arrays of COMPUTE_ROLES (kernel.py:134-136), each
//    (ncols, nz) and independent — level 0 is +0.0, levels 1..nz-2 use the mid
//    formula with tzc[k], level nz-1 the top formula (kp1 operands unused);
//  * su_formula / sv_formula / sw_formula (kernel.py:73-112) as elementwise
//    kernels over 19 broadcast arguments (tcx, tcy, tzc1_k, tzc2_k and the 15
//    operands; stride 0 for a scalar, 1 for an array) and one `top` flag.
//
// The arithmetic is the shared pw_expr of pwadv_device.cuh (the reference's
// association, one IEEE operation each).
#include "pwadv_device.cuh"
#include "pwadv_internal.h"

namespace pwadv {

// role indices in COMPUTE_ROLES order:
//  0 u(-1,0)  1 u(-1,1)  2 u(0,-1)  3 u(0,0)  4 u(0,1)  5 u(1,0)
//  6 v(-1,0)  7 v(0,-1)  8 v(0,0)   9 v(0,1) 10 v(1,-1) 11 v(1,0)
// 12 w(-1,0) 13 w(0,-1) 14 w(0,0)  15 w(0,1) 16 w(1,0)
struct RolePtrs {
    const double *r[17];
};

struct FormulaArgs {
    const double *p[19];
    int64_t stride[19];
};

template <bool FMA>
__global__ void __launch_bounds__(256)
    k_compute_block(const __grid_constant__ RolePtrs R, double *su, double *sv, double *sw,
                    int64_t total, int64_t nz, double tcx, double tcy, const double *tzc1,
                    const double *tzc2)
{
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = idx % nz;
        if (k == 0) {  // compute_block leaves level 0 at zeros_like (kernel.py:151)
            su[idx] = 0.0;
            sv[idx] = 0.0;
            sw[idx] = 0.0;
            continue;
        }
        const bool top = (k == nz - 1);
        // operand (role, dk); at the top the reference passes level t for dk = +1
        // (kernel.py:156-157) and the formulas never read it
        auto op = [&](int role, int dk) -> double {
            return __ldg(R.r[role] + idx + (top && dk > 0 ? 0 : dk));
        };
        const double c1 = __ldg(tzc1 + k), c2 = __ldg(tzc2 + k);
        // operand wiring _SU_ARGS / _SV_ARGS / _SW_ARGS (kernel.py:117-128)
        su[idx] = su_formula<FMA>(tcx, tcy, c1, c2, op(3, 0), op(0, 0), op(5, 0), op(2, 0), op(4, 0),
                                  op(3, -1), op(3, 1), op(7, 0), op(10, 0), op(8, 0), op(11, 0),
                                  op(14, -1), op(16, -1), op(14, 0), op(16, 0), top);
        sv[idx] = sv_formula<FMA>(tcx, tcy, c1, c2, op(8, 0), op(6, 0), op(11, 0), op(7, 0), op(9, 0),
                                  op(8, -1), op(8, 1), op(0, 0), op(1, 0), op(3, 0), op(4, 0),
                                  op(14, -1), op(15, -1), op(14, 0), op(15, 0), top);
        sw[idx] = sw_formula<FMA>(tcx, tcy, c1, c2, op(14, 0), op(12, 0), op(16, 0), op(13, 0),
                                  op(15, 0), op(14, -1), op(14, 1), op(0, -1), op(0, 0), op(3, -1),
                                  op(3, 0), op(7, -1), op(7, 0), op(8, -1), op(8, 0), top);
    }
}

template <bool FMA>
__global__ void __launch_bounds__(256)
    k_formula(int which, const __grid_constant__ FormulaArgs A, int64_t n, int top, double *out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        double v[19];
#pragma unroll
        for (int m = 0; m < 19; ++m) v[m] = __ldg(A.p[m] + i * A.stride[m]);
        const bool t = top != 0;
        double s;
        if (which == 0)
            s = su_formula<FMA>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9], v[10],
                                v[11], v[12], v[13], v[14], v[15], v[16], v[17], v[18], t);
        else if (which == 1)
            s = sv_formula<FMA>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9], v[10],
                                v[11], v[12], v[13], v[14], v[15], v[16], v[17], v[18], t);
        else
            s = sw_formula<FMA>(v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9], v[10],
                                v[11], v[12], v[13], v[14], v[15], v[16], v[17], v[18], t);
        out[i] = s;
    }
}

static unsigned blocks_for(int64_t total)
{
    const DeviceInfo *dev = device_info();
    int64_t b = (total + 255) / 256;
    const int64_t cap = (int64_t)(dev ? dev->sms : 148) * 8;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (unsigned)b;
}

int launch_compute_block(const double *const roles[17], double *su, double *sv, double *sw,
                         int64_t ncols, int64_t nz, double tcx, double tcy, const double *tzc1,
                         const double *tzc2, bool fma, cudaStream_t s)
{
    RolePtrs R;
    for (int m = 0; m < 17; ++m) R.r[m] = roles[m];
    const int64_t total = ncols * nz;
    if (total == 0) return PWADV_OK;
    if (fma)
        k_compute_block<true><<<blocks_for(total), 256, 0, s>>>(R, su, sv, sw, total, nz, tcx, tcy,
                                                                 tzc1, tzc2);
    else
        k_compute_block<false><<<blocks_for(total), 256, 0, s>>>(R, su, sv, sw, total, nz, tcx, tcy,
                                                                  tzc1, tzc2);
    count_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PWADV_OK : set_cuda_error("compute_block launch", e);
}

int launch_formula(int which, const double *const args[19], const int64_t strides[19], int64_t n,
                   int top, double *out, bool fma, cudaStream_t s)
{
    FormulaArgs A;
    for (int m = 0; m < 19; ++m) {
        A.p[m] = args[m];
        A.stride[m] = strides[m];
    }
    if (n == 0) return PWADV_OK;
    if (fma)
        k_formula<true><<<blocks_for(n), 256, 0, s>>>(which, A, n, top, out);
    else
        k_formula<false><<<blocks_for(n), 256, 0, s>>>(which, A, n, top, out);
    count_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PWADV_OK : set_cuda_error("formula launch", e);
}

}  // namespace pwadv
