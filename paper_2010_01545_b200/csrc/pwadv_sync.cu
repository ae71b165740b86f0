// pwadv_sync.cu — stream-ordered neighbour handshake for the fused multi-GPU
// steps.
//
// A fused step (K4 pushing boundary values into the neighbours' halos, or K1
// pulling its halo cells from the neighbours' fields) needs, before step k on
// rank r, that every NEIGHBOUR of r has finished step k-1: their stores into
// r's halos have landed (RAW) and they are done reading the buffers r is
// about to overwrite (WAR). Round 1 ordered this with a global one-element
// NCCL all-reduce per step. Here it is a neighbour-only handshake carried by
// the GPU front end, with no kernel and no host round trip:
//
//   signal: after step k, stream-ordered 64-bit writes of k into each
//           neighbour's flag array, at this rank's slot — remote stores over
//           NVLink into the neighbour's (CUDA-IPC-mapped) memory. The default
//           write carries a memory fence (__threadfence_system semantics,
//           scoped to the stream): step k's writes, peer stores included, are
//           visible before the flag is.
//   wait:   before step k+1, the stream waits until this rank's own flag
//           array holds >= k at every neighbour's slot (a local poll by the
//           front end), with CU_STREAM_WAIT_VALUE_FLUSH where the device
//           supports it (remote writes that reached the device are visible
//           to the work after the wait).
//
// Both are one cuStreamBatchMemOp each (up to 8 neighbours). Kernels never
// wait on other kernels, so ranks emulated as threads on one GPU (each with
// its own stream) exercise exactly this path. The reference analogue is the
// join of the engine threads in run_schedule (schedules.py:221-227).
#include <cuda.h>

#include "pwadv_internal.h"

#include <cstdlib>
#include <mutex>

namespace pwadv {
namespace {

typedef CUresult (*batch_fn)(CUstream, unsigned int, CUstreamBatchMemOpParams *, unsigned int);
typedef CUresult (*attr_fn)(int *, CUdevice_attribute, CUdevice);

struct DriverFns {
    batch_fn batch = nullptr;
    attr_fn attr = nullptr;
    bool ok = false;
};

const DriverFns &driver()
{
    static DriverFns d;
    static std::once_flag once;
    std::call_once(once, [] {
        void *f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuStreamBatchMemOp", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            d.batch = (batch_fn)f;
        f = nullptr;
        if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            d.attr = (attr_fn)f;
        d.ok = d.batch && d.attr;
    });
    return d;
}

// per device: 64-bit stream memory operations / remote-write flush supported
struct Caps {
    int mem64 = -1, flush = -1;
};
Caps g_caps[64];
std::mutex g_caps_mu;

int caps_of(int device, Caps *out)
{
    const DriverFns &d = driver();
    if (!d.ok) return set_error(PWADV_E_CUDA, "driver entry points for stream memory operations unavailable");
    if (device < 0 || device >= 64) return set_error(PWADV_E_ARG, "device %d out of range", device);
    std::lock_guard<std::mutex> lk(g_caps_mu);
    Caps &c = g_caps[device];
    if (c.mem64 < 0) {
        int v = 0;
        if (d.attr(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, (CUdevice)device) != CUDA_SUCCESS)
            v = 0;
        c.mem64 = v;
        v = 0;
        if (d.attr(&v, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, (CUdevice)device) != CUDA_SUCCESS) v = 0;
        c.flush = v;
    }
    *out = c;
    return PWADV_OK;
}

// nw flag writes (slots ws) then nr waits (slots rs) in ONE cuStreamBatchMemOp
int batch2(uint64_t *const *ws, int nw, uint64_t *const *rs, int nr, uint64_t value, void *stream)
{
    if (nw < 0 || nr < 0 || nw + nr > 64)
        return set_error(PWADV_E_ARG, "handshake takes 0..64 slots, got %d + %d", nw, nr);
    if (nw + nr == 0) return PWADV_OK;
    if ((nw && !ws) || (nr && !rs)) return set_error(PWADV_E_NULL, "null slots");
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_cuda_error("cudaGetDevice", e);
    Caps c;
    int rc = caps_of(dev, &c);
    if (rc) return rc;
    if (!c.mem64) return set_error(PWADV_E_CUDA, "64-bit stream memory operations unsupported on device %d", dev);
    static const bool no_flush = getenv("PWADV_HANDSHAKE_NO_FLUSH") != nullptr;  // measurement only
    CUstreamBatchMemOpParams ops[64] = {};
    for (int i = 0; i < nw + nr; ++i) {
        uint64_t *slot = i < nw ? ws[i] : rs[i - nw];
        if (!slot || ((uintptr_t)slot & 7))
            return set_error(PWADV_E_ALIGN, "handshake slot %d null or not 8-byte aligned", i);
        if (i < nw) {
            ops[i].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
            ops[i].writeValue.address = (CUdeviceptr)(uintptr_t)slot;
            ops[i].writeValue.value64 = value;
            // fenced after the preceding work (default semantics; an
            // unfenced write is rejected inside a batch)
            ops[i].writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
        } else {
            ops[i].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
            ops[i].waitValue.address = (CUdeviceptr)(uintptr_t)slot;
            ops[i].waitValue.value64 = value;
            // flush remote writes once, after the last wait
            const bool last = i == nw + nr - 1;
            ops[i].waitValue.flags =
                CU_STREAM_WAIT_VALUE_GEQ | (c.flush && last && !no_flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0);
        }
    }
    const CUresult r = driver().batch((CUstream)stream, (unsigned)(nw + nr), ops, 0);
    if (r != CUDA_SUCCESS)
        return set_error(PWADV_E_CUDA, "cuStreamBatchMemOp (%d writes, %d waits) failed: CUresult %d", nw, nr,
                         (int)r);
    return PWADV_OK;
}

// ---------------------------------------------------------------------------
// The handshake as one tiny kernel (1 CTA of 32 threads), chained to the step
// kernels by programmatic dependent launch instead of front-end memory ops:
//
//   griddepcontrol.wait — the step kernel before it has completed and its
//       writes (peer stores included) are visible;
//   lane i < nsig: st.release.sys of `value` into neighbour i's slot (a
//       remote store over NVLink; release at system scope is cumulative over
//       the step's writes this grid observed);
//   lane i < nwait: ld.acquire.sys poll of my slot for neighbour i until it
//       holds >= value (or the timeout: the error word is set and the lane
//       gives up, so a lost signal can never hang the stream);
//   griddepcontrol.launch_dependents only after every lane is done — the
//       next step kernel is launched early (PDL) but cannot take SMs while
//       the handshake still waits (with ranks emulated on one GPU, waiting
//       step CTAs could otherwise hold every SM a neighbour needs).
struct HsArgs {
    unsigned long long *sig[32];
    const unsigned long long *wait[32];
    int nsig, nwait;
    unsigned long long value;
    unsigned long long timeout_ns;
    int *err;
};

__device__ __forceinline__ unsigned long long now_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(32) k_handshake(const __grid_constant__ HsArgs a)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int i = threadIdx.x;
    if (i < a.nsig)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a.sig[i]), "l"(a.value) : "memory");
    if (i < a.nwait) {
        const unsigned long long t0 = now_ns();
        for (;;) {
            unsigned long long v;
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a.wait[i]) : "memory");
            if ((long long)(v - a.value) >= 0) break;
            if (now_ns() - t0 > a.timeout_ns) {
                atomicExch(a.err, 1);
                break;
            }
            __nanosleep(64);
        }
    }
    __syncwarp();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

}  // namespace
}  // namespace pwadv

using namespace pwadv;

extern "C" {

int pwadv_handshake_caps(int device, int *mem64, int *flush)
{
    Caps c;
    const int rc = caps_of(device, &c);
    if (rc) return rc;
    if (mem64) *mem64 = c.mem64;
    if (flush) *flush = c.flush;
    return PWADV_OK;
}

int pwadv_signal_peers(uint64_t *const *slots, int n, uint64_t value, void *stream)
{
    return batch2(slots, n, nullptr, 0, value, stream);
}

int pwadv_wait_peers(uint64_t *const *slots, int n, uint64_t value, void *stream)
{
    return batch2(nullptr, 0, slots, n, value, stream);
}

int pwadv_handshake(uint64_t *const *signal_slots, int nsignal, uint64_t *const *wait_slots, int nwait,
                    uint64_t value, void *stream)
{
    return batch2(signal_slots, nsignal, wait_slots, nwait, value, stream);
}

int pwadv_handshake_kernel(uint64_t *const *signal_slots, int nsignal, uint64_t *const *wait_slots,
                           int nwait, uint64_t value, int *err, uint64_t timeout_ns, void *stream)
{
    if (nsignal < 0 || nwait < 0 || nsignal > 32 || nwait > 32)
        return set_error(PWADV_E_ARG, "handshake kernel takes 0..32 slots each, got %d / %d", nsignal, nwait);
    if ((nsignal && !signal_slots) || (nwait && !wait_slots) || (nwait && !err))
        return set_error(PWADV_E_NULL, "null slots or error word");
    HsArgs a = {};
    for (int i = 0; i < nsignal; ++i) {
        if (!signal_slots[i] || ((uintptr_t)signal_slots[i] & 7))
            return set_error(PWADV_E_ALIGN, "signal slot %d null or not 8-byte aligned", i);
        a.sig[i] = reinterpret_cast<unsigned long long *>(signal_slots[i]);
    }
    for (int i = 0; i < nwait; ++i) {
        if (!wait_slots[i] || ((uintptr_t)wait_slots[i] & 7))
            return set_error(PWADV_E_ALIGN, "wait slot %d null or not 8-byte aligned", i);
        a.wait[i] = reinterpret_cast<const unsigned long long *>(wait_slots[i]);
    }
    a.nsig = nsignal;
    a.nwait = nwait;
    a.value = value;
    a.timeout_ns = timeout_ns ? timeout_ns : 10000000000ull;
    a.err = err;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = (cudaStream_t)stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    static const bool no_pdl = getenv("PWADV_HANDSHAKE_NO_PDL") != nullptr;  // measurement only
    cfg.numAttrs = no_pdl ? 0 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k_handshake, a);
    if (e != cudaSuccess) return set_cuda_error("handshake kernel launch", e);
    count_launch();
    return PWADV_OK;
}

}  // extern "C"
