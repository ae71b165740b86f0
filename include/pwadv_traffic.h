/*
 * pwadv_traffic.h — live DRAM traffic of the PW-advection launches
 * (libpwadv_traffic.so, optional; CUPTI range profiler).
 *
 * Replaces, for the GPU, the reference's per-run traffic counters
 * (TrafficReport, pkg/src/pwadvect/schedules.py:99-114): where the reference
 * counts the float64 elements its schedules move, these count the bytes the
 * kernels actually move through HBM (dram__bytes_read.sum /
 * dram__bytes_write.sum) plus their summed duration (gpu__time_duration.sum).
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

int pwadv_traffic_begin(int device);
/* out[0] DRAM bytes read, out[1] DRAM bytes written, out[2] kernel ns */
int pwadv_traffic_end(double out[3], int *nranges);
const char *pwadv_traffic_last_error(void);
int pwadv_traffic_max_ranges(void);

#ifdef __cplusplus
}
#endif
