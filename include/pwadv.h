/*
 * pwadv.h — C ABI of the B200-native PW-advection hot path (libpwadv.so).
 *
 * This is the drop-in boundary for the reference's hot path (pwadvect 0.1.0,
 * /root/reference). The reference has no FFI of its own: its
 * interface is the Python function
 *     run_reference(fields: FieldSet, coeffs: AdvectionCoefficients) -> SourceSet
 * (pkg/src/pwadvect/kernel.py:175-185) and the dispatcher
 *     run_schedule(fields, coeffs, ScheduleSpec) -> (SourceSet, TrafficReport, wall)
 * (pkg/src/pwadvect/schedules.py:207-232). The entry points below are what a
 * ctypes/cffi binding of that interface calls; the Python mirror in
 * paper_2010_01545_b200/ (and INTEGRATION.md) shows the binding.
 *
 * Data contract (pkg/src/pwadvect/grid.py:30-130, docs/model-notes.md §1):
 *   every field is a C-order float64 array of shape (nx+2, ny+2, nz), k fastest,
 *   halo width 1 in X and Y only; flat offset of [i, j, k] = (i*(ny+2)+j)*nz + k.
 *   Outputs su/sv/sw: interior columns are written at every level (level 0 is
 *   +0.0, kernel.py:151); halo columns are never written (the caller zeroes the
 *   output buffers once, as zeros_sources does, grid.py:129-130).
 *
 * Conventions:
 *   - All functions return 0 on success or a negative PWADV_E* code; the
 *     message of the last failure on the calling thread is pwadv_last_error().
 *   - Device-pointer functions are asynchronous on `stream` (a cudaStream_t;
 *     NULL = legacy default stream) and never retain caller memory.
 *   - No global mutable state besides a lazily initialised per-device attribute
 *     cache; safe to call from several host threads on different streams/devices.
 *   - Arithmetic is bit-exact with the reference (IEEE binary64, no FMA
 *     contraction, the reference's association order)
 *     unless PWADV_FLAG_FMA is passed.
 */
#ifndef PWADV_H_
#define PWADV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PWADV_ABI_VERSION 2

enum {
    PWADV_OK = 0,
    PWADV_E_DIMS = -1,      /* nx < 1, ny < 1 or nz < 2 (grid.py:52-58 GridError) */
    PWADV_E_NULL = -2,      /* null pointer argument */
    PWADV_E_RANGE = -3,     /* sub-box outside the interior / bad slab */
    PWADV_E_CUDA = -4,      /* CUDA launch or runtime error */
    PWADV_E_ARG = -5,       /* other invalid argument (mode, tuning) */
    PWADV_E_ALIGN = -6      /* pointer not 8-byte aligned (16-byte-aligned fields take the
                               X-march's aligned form, 8-byte-aligned ones its unaligned-run
                               form) */
};

/* flags for pwadv_opts.flags */
#define PWADV_FLAG_FMA 1u           /* contract into DFMA (not bit-exact; <=1e-12 normwise) */
#define PWADV_FLAG_SIMPLE 2u        /* force the one-thread-per-point kernel */
#define PWADV_FLAG_MARCH 4u         /* force the general march K1m (no shared-memory plane ring) */
#define PWADV_FLAG_UNALIGNED 8u     /* X-march in its unaligned-run form (copies start up to one
                                       element early, scalar shared loads/stores) even where the
                                       aligned form applies; odd nz and 8-byte-aligned fields
                                       always use it */
#define PWADV_FLAG_RIM 16u          /* only the one-cell rim of the box (one launch; multi-GPU overlap) */
#define PWADV_FLAG_GENERIC 32u      /* X-march with a run-time tile layout even for nz = 64 / 128 */
#define PWADV_FLAG_L2_UNIT_HEAD 64u /* X-march: load each work unit's first two planes L2 evict_last */
#define PWADV_FLAG_NO_PDL 128u      /* X-march: ordinary launch (default: programmatic dependent launch) */
/* ablation switches for profiling only (results are NOT the PW sources):
 * skip the PW arithmetic / skip the output stores of the X-march kernel
 * (they select the run-time-layout X-march, as PWADV_FLAG_GENERIC) */
#define PWADV_FLAG_DEBUG_NO_COMPUTE 0x100u
#define PWADV_FLAG_DEBUG_NO_STORE 0x400u
/* X-march work plan: never / always (where it applies) use the spare-tail
 * plan (main chunks + tail chunks run by the spare CTAs; default: for plans
 * of short units, <= 130 planes, when it shortens the longest CTA by >= 5%) */
#define PWADV_FLAG_NO_SPARE_TAIL 0x1000u
#define PWADV_FLAG_SPARE_TAIL 0x2000u
/* Column-tile X-march (K1c: work unit = X chunk x y-strip x k-slab, one bulk
 * copy per staged column, every (k, k+1) pair on the 16-byte grid even for odd
 * nz): force it where it applies / never use it (default: the planner's
 * choice). With it, tile_j selects the slab height
 * KT = 768 / tile_j: 6 (KT 128), 8 (96), 12 (64), 16 (48) or 24 (32); odd nz
 * takes 128 or 64 only. */
#define PWADV_FLAG_CTILE 0x4000u
#define PWADV_FLAG_NO_CTILE 0x8000u

/* Optional tuning / variant selection; pass NULL for defaults. */
typedef struct pwadv_opts {
    uint32_t flags;
    int32_t tile_j;        /* columns per CTA strip for the X-march kernel (0 = auto) */
    int32_t stages;        /* smem plane-ring depth (0 = auto) */
    int32_t grid;          /* CTAs (0 = auto: SMs x resident CTAs) */
    int32_t max_threads;   /* X-march CTA thread budget: 512 (warp-specialised: 3 compute + 1
                              producer warpgroup), 384, 256, 192 or 128 (0 = auto = 512) */
    int32_t chunks;        /* > 0: every strip in this many X chunks (work unit = chunk x strip);
                              0 = auto (whole strips for the full rounds, the rest chunked) */
    void *trace;           /* profiling only: device buffer of 2x4096 u64 for CTA 0's
                              per-plane copy-issue / arrival %globaltimer stamps; NULL = off */
} pwadv_opts;

int pwadv_abi_version(void);
/* Identity of the build: 16 hex digits of the sha256 over the library's
 * sources, headers and nvcc flags (build.py), fixed at compile time. nvcc
 * object code is not bit-reproducible (per-compilation module ids), so
 * profiles are stamped with this instead of a hash of the binary. */
const char *pwadv_source_id(void);
const char *pwadv_last_error(void);

/* Launch-count instrumentation: kernels launched by this library on the
 * calling thread since the last reset (bench.py reports it as gpu_launches). */
uint64_t pwadv_launch_count(void);
void pwadv_reset_launch_count(void);

/*
 * K1 — one PW-advection evaluation, device pointers, whole interior.
 * Replaces run_reference (kernel.py:175-185) -> compute_block (:139-162) ->
 * su/sv/sw_formula (:73-112). tzc1/tzc2: device arrays of nz doubles.
 */
int pwadv_advect_f64(const double *u, const double *v, const double *w,
                     double *su, double *sv, double *sw,
                     int64_t nx, int64_t ny, int64_t nz,
                     double tcx, double tcy,
                     const double *tzc1, const double *tzc2,
                     const pwadv_opts *opts, void *stream);

/*
 * K1 on a sub-box of interior columns: i in [x_begin, x_end), j in
 * [y_begin, y_end) (1-based interior indices, as Slab in schedules.py:53-62).
 * The reference's X-slab engine (schedules.py:131-135, 194-204) is the case
 * y_begin=1, y_end=ny+1. Used for the interior/rim split of the multi-GPU
 * overlap.
 */
int pwadv_advect_box_f64(const double *u, const double *v, const double *w,
                         double *su, double *sv, double *sw,
                         int64_t nx, int64_t ny, int64_t nz,
                         double tcx, double tcy,
                         const double *tzc1, const double *tzc2,
                         int64_t x_begin, int64_t x_end, int64_t y_begin, int64_t y_end,
                         const pwadv_opts *opts, void *stream);

/* Launch plan the library would use for K1 on this box (for reports/benches). */
typedef struct pwadv_plan_info {
    int32_t kernel;        /* 1 = X-march (bulk-copy plane ring), 2 = one-thread-per-point,
                              3 = general march (register x-window, cached loads: tall
                              columns, inputs with different 16-byte phases),
                              4 = X-march with unaligned tile runs (odd nz, 8-byte-aligned
                              fields), 5 = column-tile X-march (k-slabs of
                              2 x threads_per_column levels; strips counts
                              y-strips x slabs) */
    int32_t tile_j, threads_per_column, stages, threads, grid;
    int64_t smem_bytes, strips;
    int32_t chunks;        /* X chunks of the strips after the full rounds */
    int32_t long_strips;   /* strips run as whole-X units (full rounds of the grid) */
    int32_t spare_ctas;    /* spare-tail plan: CTAs running the strips' tail chunks (0 = off);
                              then `chunks` main chunks of main_chunk_planes per strip */
    int32_t main_chunk_planes;
} pwadv_plan_info;
int pwadv_describe_plan(int64_t nx, int64_t ny, int64_t nz,
                        int64_t x_begin, int64_t x_end, int64_t y_begin, int64_t y_end,
                        const pwadv_opts *opts, int device, pwadv_plan_info *out);

/*
 * K4 — fused forward step on a sub-box: f_new = f + dt*s_f (mul then add) for
 * f in {u, v, w}, with s computed as K1 from (u, v, w). Writes interior
 * columns of u_new/v_new/w_new in the box (all levels); halos are not written
 * (wrap or exchange afterwards). No reference counterpart; the
 * composed oracle is run_reference + numpy f + dt*s + wrap_halos.
 */
int pwadv_step_box_f64(const double *u, const double *v, const double *w,
                       double *u_new, double *v_new, double *w_new,
                       int64_t nx, int64_t ny, int64_t nz,
                       double tcx, double tcy,
                       const double *tzc1, const double *tzc2, double dt,
                       int64_t x_begin, int64_t x_end, int64_t y_begin, int64_t y_end,
                       const pwadv_opts *opts, void *stream);

/*
 * K4 with the halo exchange fused in (multi-GPU time stepping, SURVEY.md §8e
 * and §8f1): computes the whole local interior like pwadv_step_box_f64 AND
 * stores every boundary value of u_new/v_new/w_new into the halo cells of the
 * neighbouring blocks' NEW buffers that mirror it (x/y faces and corners), so
 * after one barrier across ranks every block's halos equal the periodic wrap of
 * the global fields — no separate exchange. Peer buffers are device memory
 * this GPU can store to: the same device, or another GPU's allocation opened
 * with pwadv_ipc_open (CUDA IPC, NVLink P2P). A neighbour that is this block
 * itself (an undivided axis) is given as its own buffers. Peer buffers must be
 * 8-byte aligned (PWADV_E_ALIGN otherwise); when any of them is not 16-byte
 * aligned the kernel takes its unaligned-run form, whose boundary stores are
 * 8 bytes wide. The pull entry points (below) need 16-byte-aligned peers.
 */
enum {
    PWADV_NB_XM = 0, PWADV_NB_XP = 1, PWADV_NB_YM = 2, PWADV_NB_YP = 3,
    PWADV_NB_XMYM = 4, PWADV_NB_XMYP = 5, PWADV_NB_XPYM = 6, PWADV_NB_XPYP = 7
};
typedef struct pwadv_peers {
    double *u[8], *v[8], *w[8];  /* neighbour d's new u, v, w (padded layout) */
    int64_t nx[8], ny[8];        /* neighbour d's local interior extents */
} pwadv_peers;
int pwadv_step_push_f64(const double *u, const double *v, const double *w,
                        double *u_new, double *v_new, double *w_new,
                        int64_t nx, int64_t ny, int64_t nz,
                        double tcx, double tcy,
                        const double *tzc1, const double *tzc2, double dt,
                        const pwadv_peers *peers, const pwadv_opts *opts, void *stream);

/*
 * K1 with the halo exchange fused in (pull): su, sv, sw of this block's whole
 * interior, with every halo cell the stencil reads loaded from the
 * neighbours' CURRENT u, v, w (src: the same peer table layout, extents as
 * above) instead of this block's halos — x-halo planes from the x neighbours'
 * last / first interior plane, y-halo columns from the y neighbours', the
 * corners u(0, ny+1) and v(nx+1, 0) from the diagonal ones: the values a
 * two-phase periodic exchange (wrap_halos, grid.py:203-208) would have put
 * there, so the result is bit-identical to exchange-then-pwadv_advect_f64.
 * This block's halos are neither read nor written. The neighbours' interiors
 * must be final when the kernel runs (one cross-rank barrier before the call
 * when they change). Peer buffers 16-byte aligned; needs the aligned X-march
 * (even nz <= 768, 16-byte-aligned fields), else PWADV_E_ARG. An undivided
 * axis passes this block's own buffers as its neighbours (periodic wrap with
 * no halo copy).
 */
int pwadv_advect_pull_f64(const double *u, const double *v, const double *w,
                          double *su, double *sv, double *sw,
                          int64_t nx, int64_t ny, int64_t nz,
                          double tcx, double tcy,
                          const double *tzc1, const double *tzc2,
                          const pwadv_peers *src, const pwadv_opts *opts, void *stream);

/* K4 with the halo pull: as pwadv_step_f64 over the whole interior, halos
 * loaded from src as in pwadv_advect_pull_f64; the new buffers' halos are not
 * written (the next step pulls again). */
int pwadv_step_pull_f64(const double *u, const double *v, const double *w,
                        double *u_new, double *v_new, double *w_new,
                        int64_t nx, int64_t ny, int64_t nz,
                        double tcx, double tcy,
                        const double *tzc1, const double *tzc2, double dt,
                        const pwadv_peers *src, const pwadv_opts *opts, void *stream);

/*
 * K2p — the halo exchange as one gather kernel: every halo cell of this
 * block's u, v, w (x-halo planes, y-halo columns, the four corner columns)
 * loaded from the neighbours' CURRENT interiors in `src` (peer loads over
 * NVLink for another GPU's block) — the cells a two-phase periodic exchange
 * (the reference's wrap_halos, grid.py:203-208) delivers; an undivided axis
 * names this block itself. For decomposed blocks off the aligned X-march
 * (deep columns on K1c, odd nz, 8-byte-aligned fields), where the fused pull
 * of pwadv_advect_pull_f64 does not apply: gather, then pwadv_advect_f64 /
 * pwadv_step_f64 with the planner's kernel. Writes only this block's halos and
 * reads only interiors, so neighbouring blocks may gather concurrently; the
 * neighbours' interiors must be final (one handshake before the call).
 * Buffers 8-byte aligned.
 */
int pwadv_pull_halos_f64(double *u, double *v, double *w,
                         int64_t nx, int64_t ny, int64_t nz,
                         const pwadv_peers *src, void *stream);

/* CUDA IPC helpers for the peer buffers of pwadv_step_push_f64 (one process
 * per GPU): export a device allocation (handle: 64 opaque bytes, plus the
 * pointer's byte offset inside its allocation), open a peer's export, close. */
int pwadv_ipc_export(const void *dev_ptr, unsigned char handle[64], uint64_t *offset);
int pwadv_ipc_open(const unsigned char handle[64], uint64_t offset, void **dev_ptr);
int pwadv_ipc_close(void *dev_ptr, uint64_t offset);

/*
 * Neighbour handshake for the fused multi-GPU steps (pwadv_sync.cu): before
 * step k+1 every neighbour must have finished step k (its stores into my
 * halos landed; it is done reading what I overwrite). Replaces a global
 * barrier per step with stream-ordered flag writes and waits carried by the
 * GPU front end (no kernel, no host round trip). Each rank owns a zeroed
 * device array of one uint64 slot per rank, mapped into its neighbours with
 * pwadv_ipc_open.
 *   pwadv_signal_peers: after the preceding work on `stream` (fenced), write
 *     `value` to each of slots[0..n) — my slot in each neighbour's array.
 *   pwadv_wait_peers: later work on `stream` waits until each of slots[0..n)
 *     — the neighbours' slots in my own array — holds >= value.
 * pwadv_handshake_caps reports 64-bit stream memory-op and remote-write
 * flush support (both are required / used when present). n <= 64.
 */
int pwadv_handshake_caps(int device, int *mem64, int *flush);
int pwadv_signal_peers(uint64_t *const *slots, int n, uint64_t value, void *stream);
int pwadv_wait_peers(uint64_t *const *slots, int n, uint64_t value, void *stream);
/* signal then wait, one batch of stream memory operations */
int pwadv_handshake(uint64_t *const *signal_slots, int nsignal, uint64_t *const *wait_slots,
                    int nwait, uint64_t value, void *stream);
/* the same handshake as one 32-thread kernel chained to the step kernels by
 * programmatic dependent launch (the per-step call of decomp.FlagHandshake):
 * release stores of `value` to the signal slots, acquire polls of the wait
 * slots; a poll that exceeds timeout_ns (0 = 10 s) sets *err (device int) to 1
 * and gives up, so a lost signal never hangs the stream. <= 32 slots each. */
int pwadv_handshake_kernel(uint64_t *const *signal_slots, int nsignal,
                           uint64_t *const *wait_slots, int nwait, uint64_t value, int *err,
                           uint64_t timeout_ns, void *stream);

/*
 * K6 — the reference's array-level entry points (device pointers):
 * compute_block (kernel.py:139-162): roles[17] are the COMPUTE_ROLES arrays
 * (kernel.py:134-136, sorted (field, dx, dy) order: u(-1,0) u(-1,1) u(0,-1)
 * u(0,0) u(0,1) u(1,0) v(-1,0) v(0,-1) v(0,0) v(0,1) v(1,-1) v(1,0) w(-1,0)
 * w(0,-1) w(0,0) w(0,1) w(1,0)), each ncols contiguous columns of nz levels;
 * su/sv/sw get level 0 = +0.0, the mid formula at 1..nz-2 and the top formula
 * at nz-1, exactly as compute_block. flags: PWADV_FLAG_FMA or 0.
 */
int pwadv_compute_block_f64(const double *const *roles, double *su, double *sv, double *sw,
                            int64_t ncols, int64_t nz, double tcx, double tcy,
                            const double *tzc1, const double *tzc2, uint32_t flags, void *stream);
/*
 * su_formula / sv_formula / sw_formula (kernel.py:73-112; which = 0 / 1 / 2)
 * elementwise over n points: args[19] = tcx, tcy, tzc1_k, tzc2_k and the 15
 * operands in the reference's parameter order, each read at index i*stride
 * (stride 0 = a broadcast scalar, 1 = an array); top selects the k = nz
 * branch for all points.
 */
int pwadv_formula_f64(int32_t which, const double *const *args, const int64_t *strides, int64_t n,
                      int32_t top, double *out, uint32_t flags, void *stream);

/* K2 — periodic halo wrap in place (grid.py:203-208: X then Y semantics). */
int pwadv_wrap_halos_f64(double *f, int64_t nx, int64_t ny, int64_t nz, void *stream);
/* K2 on three fields in one launch. */
int pwadv_wrap_halos3_f64(double *u, double *v, double *w,
                          int64_t nx, int64_t ny, int64_t nz, void *stream);

/*
 * K5 — device field generator (grid.py:133-239), bit-identical to the
 * reference's fill_fields. Fills the interiors of u, v, w and wraps halos.
 *   mode 0: GeneratorSpec.random(seed): one Knuth-MMIX LCG stream, u then v
 *           then w interior in C order, value (state>>11)*2^-53.
 *   mode 1: BASELINE.json distribution: mode 0 value x mapped
 *           to x*20.0-10.0 (no FMA); w = 0 at levels 0 and nz-1.
 *   mode 2: GeneratorSpec.uniform(a, b, c): u=a, v=b, w=c everywhere.
 */
int pwadv_fill_f64(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                   int32_t mode, uint64_t seed, double a, double b, double c, void *stream);

/* K5 on one block of an x-y decomposition: fills the interior columns of the
 * local (nx, ny, nz) arrays with global columns (x_off+1 .. x_off+nx,
 * y_off+1 .. y_off+ny) of the (gnx, gny, nz) grid's stream. Halos are left
 * for the halo exchange. */
int pwadv_fill_box_f64(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                       int64_t gnx, int64_t gny, int64_t x_off, int64_t y_off, int32_t mode,
                       uint64_t seed, double a, double b, double c, void *stream);

/* Halo exchange helpers (multi-GPU x-y decomposition).
 * Y faces are (nx+2) runs of nz doubles at stride (ny+2)*nz: pack the column
 * j (all i in 0..nx+1) of u, v, w into buf[3][nx+2][nz], or unpack into it. */
int pwadv_pack_yface3_f64(const double *u, const double *v, const double *w, double *buf,
                          int64_t nx, int64_t ny, int64_t nz, int64_t j, void *stream);
int pwadv_unpack_yface3_f64(double *u, double *v, double *w, const double *buf,
                            int64_t nx, int64_t ny, int64_t nz, int64_t j, void *stream);
/* X faces: plane i (all j in 0..ny+1) of u, v, w <-> buf[3][ny+2][nz]. */
int pwadv_pack_xface3_f64(const double *u, const double *v, const double *w, double *buf,
                          int64_t nx, int64_t ny, int64_t nz, int64_t i, void *stream);
int pwadv_unpack_xface3_f64(double *u, double *v, double *w, const double *buf,
                            int64_t nx, int64_t ny, int64_t nz, int64_t i, void *stream);
/* Both faces of one axis in one launch (the exchange's per-axis step):
 * pack: interior face 1 -> buf_lo, face n -> buf_hi (n = nx for axis 0,
 * ny for axis 1; buffers as above); unpack: buf_lo -> halo 0, buf_hi ->
 * halo n+1. */
int pwadv_pack_faces3_f64(const double *u, const double *v, const double *w, double *buf_lo,
                          double *buf_hi, int64_t nx, int64_t ny, int64_t nz, int32_t axis,
                          void *stream);
int pwadv_unpack_faces3_f64(double *u, double *v, double *w, const double *buf_lo,
                            const double *buf_hi, int64_t nx, int64_t ny, int64_t nz, int32_t axis,
                            void *stream);
/* Local periodic copy of one axis (an undivided axis of the decomposition):
 * axis 0 = X faces (planes), axis 1 = Y faces (columns, all i incl. halos). */
int pwadv_wrap_axis3_f64(double *u, double *v, double *w, int64_t nx, int64_t ny, int64_t nz,
                         int32_t axis, void *stream);

/*
 * Host-buffer entry (end-to-end drop-in): u/v/w/su/sv/sw/tzc1/tzc2 are HOST
 * pointers (pinned or pageable). The context owns device buffers for one grid
 * shape and three streams; the call pipelines X-slab chunks so the H2D copy of
 * chunk c+1, the K1 launch on chunk c and the D2H copy of chunk c-1 overlap
 * (the paper's proposed future work). Synchronous: returns after
 * the outputs are in host memory. Output halos and level 0 are +0.0.
 * chunks <= 0 picks the count automatically (1 for fields under 32 MiB, else 16;
 * for pwadv_ctx_submit_host about 64 MiB per field and chunk, at most 16).
 */
/* A context serves one call at a time (its device buffers and streams are
 * shared by its calls); use one context per host thread for concurrency. */
typedef struct pwadv_ctx pwadv_ctx;
int pwadv_ctx_create(pwadv_ctx **out, int device, int64_t nx, int64_t ny, int64_t nz);
int pwadv_ctx_destroy(pwadv_ctx *ctx);
int pwadv_ctx_advect_host(pwadv_ctx *ctx,
                          const double *u, const double *v, const double *w,
                          double *su, double *sv, double *sw,
                          double tcx, double tcy, const double *tzc1, const double *tzc2,
                          int32_t chunks, const pwadv_opts *opts);
/* Asynchronous form for streams of grids (page-locked host buffers only):
 * enqueues one evaluation exactly like pwadv_ctx_advect_host and returns;
 * consecutive submissions alternate between two device buffer sets so the H2D
 * of one overlaps the K1/D2H of the previous. Host buffers must stay valid
 * until pwadv_ctx_sync returns (it waits for every submission). */
int pwadv_ctx_submit_host(pwadv_ctx *ctx,
                          const double *u, const double *v, const double *w,
                          double *su, double *sv, double *sw,
                          double tcx, double tcy, const double *tzc1, const double *tzc2,
                          int32_t chunks, const pwadv_opts *opts);
int pwadv_ctx_sync(pwadv_ctx *ctx);
/* Bytes moved host->device and device->host by the last ctx_advect_host call. */
int pwadv_ctx_last_bytes(const pwadv_ctx *ctx, uint64_t *h2d, uint64_t *d2h);

#ifdef __cplusplus
}
#endif
#endif /* PWADV_H_ */
