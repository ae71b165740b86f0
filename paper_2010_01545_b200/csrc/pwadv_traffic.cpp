// pwadv_traffic.cpp — live DRAM traffic of the PW-advection launches from the
// hardware counters (libpwadv_traffic.so).
//
// The reference reports element traffic for every run (TrafficReport,
// pkg/src/pwadvect/schedules.py:99-114). On the GPU the bytes that matter are
// the ones the launches move through HBM; this library reads them from the
// performance counters with the CUPTI range profiler: between
// pwadv_traffic_begin() and pwadv_traffic_end() every kernel launched on the
// current CUDA context is one auto-range (kernel replay, so multi-pass
// metric sets still need no cooperation from the caller), and end() sums
// dram__bytes_read.sum, dram__bytes_write.sum and gpu__time_duration.sum over
// the ranges. Separate from libpwadv.so so the compute library does not
// depend on libcupti; profiling is a diagnostic, never on the timed path.
//
// Not thread-safe across concurrent sessions: one session per process at a
// time (the range profiler owns the context while enabled).

#include <cuda.h>
#include <cupti_profiler_host.h>
#include <cupti_profiler_target.h>
#include <cupti_range_profiler.h>
#include <cupti_target.h>

#include "../../include/pwadv_traffic.h"

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace {

// out[] order of pwadv_traffic_end; the fp64-pipe percentage is combined over
// ranges weighted by each range's duration, the other values are summed
const char *kMetrics[] = {"dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                          "sm__inst_executed_pipe_fp64.sum"};
constexpr size_t kTimeMetric = 2, kPctMetric = 3;
constexpr size_t kNumMetrics = sizeof(kMetrics) / sizeof(kMetrics[0]);
constexpr size_t kMaxRanges = 256;
static_assert(kNumMetrics == PWADV_TRAFFIC_NVALUES, "pwadv_traffic.h out[] layout");

thread_local char g_err[512];

int fail(const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return -1;
}

const char *cupti_msg(CUptiResult r)
{
    const char *s = nullptr;
    cuptiGetResultString(r, &s);
    return s ? s : "unknown CUPTI error";
}

struct Session {
    bool active = false;
    CUcontext ctx = nullptr;
    CUpti_Profiler_Host_Object *host = nullptr;
    CUpti_RangeProfiler_Object *prof = nullptr;
    std::vector<uint8_t> config, counters;
};

std::mutex g_mu;
Session g_s;
bool g_cupti_init = false;

#define CUPTI_TRY(call)                                                          \
    do {                                                                         \
        CUptiResult _r = (call);                                                 \
        if (_r != CUPTI_SUCCESS) return fail("%s: %s", #call, cupti_msg(_r));     \
    } while (0)

void teardown(Session &s)
{
    if (s.prof) {
        CUpti_RangeProfiler_Disable_Params d{CUpti_RangeProfiler_Disable_Params_STRUCT_SIZE};
        d.pRangeProfilerObject = s.prof;
        cuptiRangeProfilerDisable(&d);
        s.prof = nullptr;
    }
    if (s.host) {
        CUpti_Profiler_Host_Deinitialize_Params d{CUpti_Profiler_Host_Deinitialize_Params_STRUCT_SIZE};
        d.pHostObject = s.host;
        cuptiProfilerHostDeinitialize(&d);
        s.host = nullptr;
    }
    s.active = false;
}

int begin_locked(int device)
{
    if (cuInit(0) != CUDA_SUCCESS) return fail("cuInit failed");
    CUcontext ctx = nullptr;
    cuCtxGetCurrent(&ctx);
    if (!ctx) {  // the runtime's primary context of `device`
        CUdevice dev;
        if (cuDeviceGet(&dev, device) != CUDA_SUCCESS) return fail("no CUDA device %d", device);
        if (cuDevicePrimaryCtxRetain(&ctx, dev) != CUDA_SUCCESS || cuCtxSetCurrent(ctx) != CUDA_SUCCESS)
            return fail("cannot make the primary context of device %d current", device);
    }
    CUdevice cur;
    if (cuCtxGetDevice(&cur) != CUDA_SUCCESS) return fail("cuCtxGetDevice failed");
    if (!g_cupti_init) {
        CUpti_Profiler_Initialize_Params ip{CUpti_Profiler_Initialize_Params_STRUCT_SIZE};
        CUPTI_TRY(cuptiProfilerInitialize(&ip));
        g_cupti_init = true;
    }
    CUpti_Profiler_DeviceSupported_Params sup{CUpti_Profiler_DeviceSupported_Params_STRUCT_SIZE};
    sup.cuDevice = cur;
    sup.api = CUPTI_PROFILER_RANGE_PROFILING;
    CUPTI_TRY(cuptiProfilerDeviceSupported(&sup));
    if (sup.isSupported != CUPTI_PROFILER_CONFIGURATION_SUPPORTED)
        return fail("range profiling not supported on device %d (vGPU/confidential compute/arch)", (int)cur);

    Session &s = g_s;
    s.ctx = ctx;
    // chip + counter availability -> host object -> config image of the metrics
    CUpti_Device_GetChipName_Params cn{CUpti_Device_GetChipName_Params_STRUCT_SIZE};
    cn.deviceIndex = (size_t)cur;
    CUPTI_TRY(cuptiDeviceGetChipName(&cn));
    CUpti_Profiler_GetCounterAvailability_Params av{CUpti_Profiler_GetCounterAvailability_Params_STRUCT_SIZE};
    av.ctx = ctx;
    CUPTI_TRY(cuptiProfilerGetCounterAvailability(&av));
    std::vector<uint8_t> avail(av.counterAvailabilityImageSize);
    av.pCounterAvailabilityImage = avail.data();
    CUPTI_TRY(cuptiProfilerGetCounterAvailability(&av));

    CUpti_Profiler_Host_Initialize_Params hi{CUpti_Profiler_Host_Initialize_Params_STRUCT_SIZE};
    hi.profilerType = CUPTI_PROFILER_TYPE_RANGE_PROFILER;
    hi.pChipName = cn.pChipName;
    hi.pCounterAvailabilityImage = avail.data();
    CUPTI_TRY(cuptiProfilerHostInitialize(&hi));
    s.host = hi.pHostObject;

    CUpti_Profiler_Host_ConfigAddMetrics_Params am{CUpti_Profiler_Host_ConfigAddMetrics_Params_STRUCT_SIZE};
    am.pHostObject = s.host;
    am.ppMetricNames = kMetrics;
    am.numMetrics = kNumMetrics;
    CUPTI_TRY(cuptiProfilerHostConfigAddMetrics(&am));
    CUpti_Profiler_Host_GetConfigImageSize_Params cs{CUpti_Profiler_Host_GetConfigImageSize_Params_STRUCT_SIZE};
    cs.pHostObject = s.host;
    CUPTI_TRY(cuptiProfilerHostGetConfigImageSize(&cs));
    s.config.assign(cs.configImageSize, 0);
    CUpti_Profiler_Host_GetConfigImage_Params ci{CUpti_Profiler_Host_GetConfigImage_Params_STRUCT_SIZE};
    ci.pHostObject = s.host;
    ci.pConfigImage = s.config.data();
    ci.configImageSize = s.config.size();
    CUPTI_TRY(cuptiProfilerHostGetConfigImage(&ci));

    // range profiler on the context: one auto-range per kernel, kernel replay
    CUpti_RangeProfiler_Enable_Params en{CUpti_RangeProfiler_Enable_Params_STRUCT_SIZE};
    en.ctx = ctx;
    CUPTI_TRY(cuptiRangeProfilerEnable(&en));
    s.prof = en.pRangeProfilerObject;
    CUpti_RangeProfiler_GetCounterDataSize_Params ds{CUpti_RangeProfiler_GetCounterDataSize_Params_STRUCT_SIZE};
    ds.pRangeProfilerObject = s.prof;
    ds.pMetricNames = kMetrics;
    ds.numMetrics = kNumMetrics;
    ds.maxNumOfRanges = kMaxRanges;
    ds.maxNumRangeTreeNodes = kMaxRanges;
    CUPTI_TRY(cuptiRangeProfilerGetCounterDataSize(&ds));
    s.counters.assign(ds.counterDataSize, 0);
    CUpti_RangeProfiler_CounterDataImage_Initialize_Params cd{
        CUpti_RangeProfiler_CounterDataImage_Initialize_Params_STRUCT_SIZE};
    cd.pRangeProfilerObject = s.prof;
    cd.pCounterData = s.counters.data();
    cd.counterDataSize = s.counters.size();
    CUPTI_TRY(cuptiRangeProfilerCounterDataImageInitialize(&cd));
    CUpti_RangeProfiler_SetConfig_Params sc{CUpti_RangeProfiler_SetConfig_Params_STRUCT_SIZE};
    sc.pRangeProfilerObject = s.prof;
    sc.pConfig = s.config.data();
    sc.configSize = s.config.size();
    sc.pCounterDataImage = s.counters.data();
    sc.counterDataImageSize = s.counters.size();
    sc.maxRangesPerPass = kMaxRanges;
    sc.numNestingLevels = 1;
    sc.minNestingLevel = 1;
    sc.passIndex = 0;
    sc.targetNestingLevel = 1;
    sc.range = CUPTI_AutoRange;
    sc.replayMode = CUPTI_KernelReplay;
    CUPTI_TRY(cuptiRangeProfilerSetConfig(&sc));
    CUpti_RangeProfiler_Start_Params st{CUpti_RangeProfiler_Start_Params_STRUCT_SIZE};
    st.pRangeProfilerObject = s.prof;
    CUPTI_TRY(cuptiRangeProfilerStart(&st));
    // auto ranges are taken only for kernels inside a pushed range of the
    // target nesting level: one enclosing range for the whole session
    CUpti_RangeProfiler_PushRange_Params pr{CUpti_RangeProfiler_PushRange_Params_STRUCT_SIZE};
    pr.pRangeProfilerObject = s.prof;
    pr.pRangeName = "pwadv";
    CUPTI_TRY(cuptiRangeProfilerPushRange(&pr));
    s.active = true;
    return 0;
}

int end_locked(double *out, int *nranges)
{
    Session &s = g_s;
    CUpti_RangeProfiler_PopRange_Params pp{CUpti_RangeProfiler_PopRange_Params_STRUCT_SIZE};
    pp.pRangeProfilerObject = s.prof;
    CUPTI_TRY(cuptiRangeProfilerPopRange(&pp));
    CUpti_RangeProfiler_Stop_Params sp{CUpti_RangeProfiler_Stop_Params_STRUCT_SIZE};
    sp.pRangeProfilerObject = s.prof;
    CUPTI_TRY(cuptiRangeProfilerStop(&sp));
    CUpti_RangeProfiler_DecodeData_Params dd{CUpti_RangeProfiler_DecodeData_Params_STRUCT_SIZE};
    dd.pRangeProfilerObject = s.prof;
    CUPTI_TRY(cuptiRangeProfilerDecodeData(&dd));
    CUpti_RangeProfiler_GetCounterDataInfo_Params gi{CUpti_RangeProfiler_GetCounterDataInfo_Params_STRUCT_SIZE};
    gi.pCounterDataImage = s.counters.data();
    gi.counterDataImageSize = s.counters.size();
    CUPTI_TRY(cuptiRangeProfilerGetCounterDataInfo(&gi));
    if (getenv("PWADV_TRAFFIC_DEBUG"))
        fprintf(stderr, "pwadv_traffic: allpass=%d ranges=%zu counters=%zu config=%zu\n",
                (int)sp.isAllPassSubmitted, (size_t)gi.numTotalRanges, s.counters.size(), s.config.size());
    for (size_t m = 0; m < kNumMetrics; ++m) out[m] = 0.0;
    for (size_t r = 0; r < gi.numTotalRanges; ++r) {
        double v[kNumMetrics] = {};
        CUpti_Profiler_Host_EvaluateToGpuValues_Params ev{
            CUpti_Profiler_Host_EvaluateToGpuValues_Params_STRUCT_SIZE};
        ev.pHostObject = s.host;
        ev.pCounterDataImage = s.counters.data();
        ev.counterDataImageSize = s.counters.size();
        ev.ppMetricNames = kMetrics;
        ev.numMetrics = kNumMetrics;
        ev.rangeIndex = r;
        ev.pMetricValues = v;
        CUPTI_TRY(cuptiProfilerHostEvaluateToGpuValues(&ev));
        for (size_t m = 0; m < kNumMetrics; ++m)
            out[m] += m == kPctMetric ? v[m] * v[kTimeMetric] : v[m];
    }
    out[kPctMetric] = out[kTimeMetric] > 0.0 ? out[kPctMetric] / out[kTimeMetric] : 0.0;
    *nranges = (int)gi.numTotalRanges;
    return 0;
}

}  // namespace

extern "C" {

// Start counting on the calling thread's current CUDA context (or device's
// primary context). Returns 0, or -1 with pwadv_traffic_last_error() set.
int pwadv_traffic_begin(int device)
{
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_s.active) return fail("a traffic session is already active");
    const int rc = begin_locked(device);
    if (rc) teardown(g_s);
    return rc;
}

// Stop counting (the caller has synchronised its launches). Over the *nranges
// kernels launched since begin: out[0] = DRAM bytes read, out[1] = DRAM bytes
// written, out[2] = summed kernel duration in ns, out[3] = fp64-pipe active
// cycles in % of peak (duration-weighted mean), out[4] = fp64 warp
// instructions executed.
int pwadv_traffic_end(double out[PWADV_TRAFFIC_NVALUES], int *nranges)
{
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_s.active) return fail("no active traffic session");
    if (!out || !nranges) {
        teardown(g_s);
        return fail("null argument");
    }
    const int rc = end_locked(out, nranges);
    teardown(g_s);
    return rc;
}

const char *pwadv_traffic_last_error(void) { return g_err; }

int pwadv_traffic_max_ranges(void) { return (int)kMaxRanges; }

int pwadv_traffic_num_values(void) { return (int)kNumMetrics; }

}  // extern "C"
