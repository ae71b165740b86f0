/*
 * pwadv_traffic.h — live DRAM traffic of the PW-advection launches
 * (libpwadv_traffic.so, optional; CUPTI range profiler).
 *
 * Replaces, for the GPU, the reference's per-run traffic counters
 * (TrafficReport, pkg/src/pwadvect/schedules.py:99-114): where the reference
 * counts the float64 elements its schedules move, these count the bytes the
 * kernels actually move through HBM (dram__bytes_read.sum /
 * dram__bytes_write.sum) plus their summed duration (gpu__time_duration.sum)
 * and the fp64-pipe utilisation the north star asks the harness to report.
 *
 * Usage: pwadv_traffic_begin(device); launch; cudaDeviceSynchronize();
 * pwadv_traffic_end(out, &n). Every kernel launched on the current context in
 * between is one range (kernel replay); the values are summed over the n
 * ranges (at most pwadv_traffic_max_ranges()). One session per process at a
 * time. Diagnostic only: never inside a timed region.
 */
#pragma once
#ifdef __cplusplus
extern "C" {
#endif

#define PWADV_TRAFFIC_NVALUES 5

int pwadv_traffic_begin(int device);
/* out[0] DRAM bytes read, out[1] DRAM bytes written, out[2] kernel ns (all
 * summed over the ranges), out[3] fp64-pipe active cycles in % of peak
 * (sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active, mean
 * weighted by range duration), out[4] fp64 warp instructions
 * (sm__inst_executed_pipe_fp64.sum) */
int pwadv_traffic_end(double out[PWADV_TRAFFIC_NVALUES], int *nranges);
const char *pwadv_traffic_last_error(void);
int pwadv_traffic_max_ranges(void);
int pwadv_traffic_num_values(void); /* PWADV_TRAFFIC_NVALUES of this build */

#ifdef __cplusplus
}
#endif
