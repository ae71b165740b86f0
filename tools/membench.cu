// membench.cu — calibration kernels for the HBM roofline of a 3-in/3-out
// stream (the PW path's traffic shape). Profiling aid, not part of libpwadv.
#include <cstdint>
#include <cuda_runtime.h>

__global__ void copy3(const double2 *__restrict__ a, const double2 *__restrict__ b,
                      const double2 *__restrict__ c, double2 *x, double2 *y, double2 *z, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double2 p = __ldg(a + i), q = __ldg(b + i), r = __ldg(c + i);
        __stcs(x + i, p);
        __stcs(y + i, q);
        __stcs(z + i, r);
    }
}

__global__ void copy1(const double2 *__restrict__ a, double2 *x, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        __stcs(x + i, __ldg(a + i));
}

__global__ void read3(const double2 *__restrict__ a, const double2 *__restrict__ b,
                      const double2 *__restrict__ c, double *sink, int64_t n)
{
    double s = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double2 p = __ldg(a + i), q = __ldg(b + i), r = __ldg(c + i);
        s += p.x + q.y + r.x;
    }
    if (s == 12345.678) sink[0] = s;
}

__global__ void write3(double2 *x, double2 *y, double2 *z, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double2 v = make_double2((double)i, 1.0);
        __stcs(x + i, v);
        __stcs(y + i, v);
        __stcs(z + i, v);
    }
}

extern "C" int mb_run(int which, void *const *in, void *const *out, int64_t n2, int grid, int block,
                      void *stream)
{
    cudaStream_t s = (cudaStream_t)stream;
    const double2 *a = (const double2 *)in[0], *b = (const double2 *)in[1], *c = (const double2 *)in[2];
    double2 *x = (double2 *)out[0], *y = (double2 *)out[1], *z = (double2 *)out[2];
    switch (which) {
    case 0: copy3<<<grid, block, 0, s>>>(a, b, c, x, y, z, n2); break;
    case 1: copy1<<<grid, block, 0, s>>>(a, x, n2); break;
    case 2: read3<<<grid, block, 0, s>>>(a, b, c, (double *)x, n2); break;
    case 3: write3<<<grid, block, 0, s>>>(x, y, z, n2); break;
    default: return -1;
    }
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}

// ---------------------------------------------------------------------------
// Staging-path calibration: each CTA streams a contiguous region of `a`
// through a shared-memory ring of `stages` x `chunk` bytes. mode 0: one
// cp.async.bulk per chunk (TMA engine), issued by thread 0, completion on an
// mbarrier; mode 1: cp.async 16-byte copies by all threads (LDGSTS);
// mode 2: LDG.128 + STS by all threads. A trivial consumer reads one value.
__device__ __forceinline__ uint32_t s32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void stage_bench(const char *__restrict__ a, int64_t bytes_per_cta, int chunk, int stages,
                            int mode, double *sink)
{
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *bar = (uint64_t *)(sm + (size_t)stages * chunk);
    const char *src = a + (int64_t)blockIdx.x * bytes_per_cta;
    const int nchunks = (int)(bytes_per_cta / chunk);
    double acc = 0;
    if (mode == 0) {
        if (threadIdx.x == 0) {
            for (int s = 0; s < stages; ++s)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar[s])));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            for (int q = 0; q < stages && q < nchunks; ++q) {
                asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[q])), "r"(chunk) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(s32(sm + (size_t)q * chunk)), "l"(src + (int64_t)q * chunk), "r"(chunk), "r"(s32(&bar[q])) : "memory");
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int q = 0; q < nchunks; ++q) {
                const int st = q % stages;
                const uint32_t par = (q / stages) & 1;
                asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P1, [%0], %1;\n@!P1 bra.uni W_%=;\n}\n" ::"r"(s32(&bar[st])), "r"(par) : "memory");
                acc += *(const double *)(sm + (size_t)st * chunk);
                const int nq = q + stages;
                if (nq < nchunks) {
                    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar[st])), "r"(chunk) : "memory");
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                 ::"r"(s32(sm + (size_t)st * chunk)), "l"(src + (int64_t)nq * chunk), "r"(chunk), "r"(s32(&bar[st])) : "memory");
                }
            }
        }
    } else {
        const int per = chunk / 16;
        for (int q = 0; q < nchunks + stages - 1; ++q) {
            if (q < nchunks) {
                const int st = q % stages;
                for (int e = threadIdx.x; e < per; e += blockDim.x) {
                    const char *g = src + (int64_t)q * chunk + e * 16;
                    unsigned char *d = sm + (size_t)st * chunk + e * 16;
                    if (mode == 1) {
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s32(d)), "l"(g) : "memory");
                    } else {
                        *(double2 *)d = __ldg((const double2 *)g);
                    }
                }
                if (mode == 1) asm volatile("cp.async.commit_group;" ::: "memory");
            }
            if (q >= stages - 1) {
                if (mode == 1) asm volatile("cp.async.wait_group %0;" ::"n"(0) : "memory");
                __syncthreads();
                acc += *(const double *)(sm + (size_t)((q - stages + 1) % stages) * chunk + threadIdx.x * 8);
                __syncthreads();
            }
        }
    }
    if (acc == 1234.5) sink[0] = acc;
}

extern "C" int mb_stage(const void *a, int64_t bytes_per_cta, int chunk, int stages, int mode, int grid,
                        int block, void *sink, void *stream)
{
    size_t smem = (size_t)stages * chunk + stages * 8;
    cudaFuncSetAttribute(stage_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    stage_bench<<<grid, block, smem, (cudaStream_t)stream>>>((const char *)a, bytes_per_cta, chunk, stages,
                                                             mode, (double *)sink);
    return cudaGetLastError() == cudaSuccess ? 0 : -2;
}
