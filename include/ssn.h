/*
 * ssn.h — C-ABI of the B200-native SubNetAct execution engine.
 *
 * The reference (servesim, C++20 header-only) models the SubNetAct worker
 * data plane only as arithmetic: a worker thread pops a
 * `DispatchCmd{batch, subnet_index, sleep_us}` and sleeps
 * (reference proj/include/servesim/serve_runtime.hpp:99-104, 161-172, sleep at
 * :167), and the simulator charges `completion = now + actuation + l_phi(B)`
 * (simcore.hpp:246-252).  This library is what a worker calls INSTEAD of that
 * sleep: `ssn_actuate(subnet_index)` + `ssn_forward(batch)`.  See
 * INTEGRATION.md for the worker-side binding.
 *
 * Conventions (mirroring the reference's error behaviour, profile.hpp:40-53,
 * policy.hpp:92-98): every entry point returns 0 on success or a negative
 * SSN_E* code; the message of the last failure on the calling thread is
 * available from ssn_last_error().  The C++ wrapper (ssn.hpp) rethrows these
 * as std::invalid_argument / std::out_of_range / std::runtime_error exactly
 * where the reference throws.
 *
 * Threading: one engine per GPU, driven by exactly one worker thread
 * (reference serve_runtime.hpp:1-6 — the dispatcher never touches workers'
 * state).  No entry point allocates device memory after ssn_prepare().
 */
#ifndef SSN_H
#define SSN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define SSN_OK 0
#define SSN_E_INVALID (-1)   /* std::invalid_argument in the reference   */
#define SSN_E_RANGE (-2)     /* std::out_of_range (unknown id / batch)    */
#define SSN_E_CUDA (-3)      /* CUDA runtime / driver failure             */
#define SSN_E_STATE (-4)     /* std::logic_error: call order violated     */
#define SSN_E_NOMEM (-5)

/* ---- supernet families --------------------------------------------------- */
enum ssn_family {
  SSN_FAMILY_TINYCNN = 1,       /* BASELINE config 1      */
  SSN_FAMILY_OFA_RESNET50 = 2,  /* BASELINE config 2      */
  SSN_FAMILY_OFA_MBV3 = 3,      /* BASELINE config 3      */
  SSN_FAMILY_BERT = 4           /* BASELINE config 5      */
};

enum ssn_dtype { SSN_DTYPE_F32 = 0, SSN_DTYPE_BF16 = 1 };

enum ssn_input_format {
  SSN_INPUT_F32_NCHW = 0, /* float32 [N][3][H][W]                          */
  SSN_INPUT_U8_NHWC = 1   /* uint8 [N][H][W][3]; value = (u8 - 128) / 64   */
};

typedef struct ssn_supernet_desc {
  uint32_t family;       /* enum ssn_family                                */
  uint32_t dtype;        /* enum ssn_dtype: storage/compute precision      */
  uint32_t image_size;   /* H == W of the input images                    */
  uint32_t num_classes;  /* classifier width                               */
  uint32_t max_batch;    /* largest batch any forward will carry           */
  uint32_t input_format; /* enum ssn_input_format                          */
  uint64_t seed;         /* weight seed when no host blob is supplied      */
  uint32_t reserved[8];
} ssn_supernet_desc;

/*
 * Subnet control tuple (D, E, W) — the C view of servesim::SubnetConfig
 * (reference profile.hpp:28-54).  Lists keep the reference's meaning:
 *   depth_flags        LayerSelect: one flag per skippable block (1 = run)
 *   expand_ratios      WeightSlice: per-block expand ratio E (> 0)
 *   width_multipliers  WeightSlice: per-stage width multiplier W in (0, 1]
 *   kernel_sizes       extension for elastic-kernel supernets (OFA-MBv3);
 *                      NULL / 0 = max kernel everywhere
 * Family-specific list lengths are documented in DESIGN.md §3.
 */
typedef struct ssn_subnet_cfg {
  const uint8_t* depth_flags;
  uint32_t n_depth;
  const double* expand_ratios;
  uint32_t n_expand;
  const double* width_multipliers;
  uint32_t n_width;
  const uint32_t* kernel_sizes;
  uint32_t n_kernel;
} ssn_subnet_cfg;

typedef struct ssn_stats {
  uint64_t weight_bytes;          /* shared weight store resident in HBM   */
  uint64_t norm_table_bytes;      /* all registered SubnetNorm rows        */
  uint64_t max_subnet_stat_bytes; /* largest single SubnetNorm row (mu,var) */
  uint64_t arena_bytes;           /* activation arena                       */
  uint32_t registered_subnets;
  int32_t active_subnet;          /* -1 before the first actuation          */
  uint32_t graphs_built;          /* LayerSelect graph segments             */
  uint32_t last_forward_kernels;  /* kernels launched by the last forward   */
  uint32_t last_forward_graphs;   /* graph segments launched                */
  uint32_t reserved0;
  double last_actuate_us;         /* host wall time of the last ssn_actuate */
  double last_forward_host_us;    /* host enqueue time of the last forward  */
} ssn_stats;

typedef struct ssn_engine ssn_engine;

/* Bytes of the host weight blob ssn_create() accepts for this descriptor
 * (layout: DESIGN.md §4 — canonical tensor order, storage layouts). */
int ssn_weight_blob_bytes(const ssn_supernet_desc* desc, uint64_t* bytes);

/* Fill a host blob from `desc->seed` with the ssn_rng.h specification. */
int ssn_generate_weight_blob(const ssn_supernet_desc* desc, void* blob,
                             uint64_t bytes);

/* SubnetNorm statistics count for a control tuple without an engine (host
 * only; same value as ssn_subnet_stat_count). Validates the tuple exactly like
 * servesim::SubnetConfig::validate (reference profile.hpp:40-53) plus the
 * supernet's max-shape bounds. */
int ssn_plan_stat_count(const ssn_supernet_desc* desc, const ssn_subnet_cfg* cfg,
                        uint64_t* count);

/* Resolved execution plan of a subnet (one row per supernet op, skipped
 * blocks marked inactive).  Used by the profiler / roofline accounting. */
typedef struct ssn_op_info {
  uint32_t kind;     /* 0 input, 1 conv, 2 maxpool, 3 avgpool, 4 gap, 5 linear */
  uint32_t active;   /* LayerSelect: 0 = block skipped                        */
  uint32_t k, stride;
  uint32_t hin, win, hout, wout;
  uint32_t cin, cout;         /* active (WeightSlice) widths                  */
  uint32_t cin_max, cout_max; /* max-shape widths                             */
  uint32_t depthwise, segment, block, has_residual;
} ssn_op_info;

int ssn_plan_ops(const ssn_supernet_desc* desc, const ssn_subnet_cfg* cfg,
                 ssn_op_info* out, uint32_t capacity, uint32_t* n_ops);

/* Build the engine on `device`: uploads the supernet weight store ONCE
 * (max-shape tensors; every subnet reads leading slices in place).
 * host_weights == NULL -> weights generated from desc->seed. */
int ssn_create(int device, const ssn_supernet_desc* desc,
               const void* host_weights, uint64_t host_weight_bytes,
               ssn_engine** out);

void ssn_destroy(ssn_engine* eng);

/* Number of SubnetNorm statistics (floats per mean / var array) the subnet
 * needs: sum of active channels over its active norm layers, in execution
 * order. */
int ssn_subnet_stat_count(ssn_engine* eng, const ssn_subnet_cfg* cfg,
                          uint64_t* count);

/* Register subnet `id` (the index into the pareto-sorted catalog, reference
 * policy.hpp:187-190) with its control tuple and SubnetNorm statistics.
 * bn_mean / bn_var == NULL -> deterministic defaults from ssn_rng.h; else both
 * must hold exactly ssn_subnet_stat_count(cfg) floats (the C-ABI cannot check
 * the length: use ssn_register_subnet_n, which takes it).
 * Folds (gamma, beta, mu_{i,j}, var_{i,j}) into per-channel scale/shift. */
int ssn_register_subnet(ssn_engine* eng, uint32_t id, const ssn_subnet_cfg* cfg,
                        const float* bn_mean, const float* bn_var);

/* Same, with the length of bn_mean / bn_var: fails with SSN_E_INVALID unless
 * n_stats == ssn_subnet_stat_count(cfg) (or both arrays are NULL), and when
 * exactly one of the two arrays is NULL. */
int ssn_register_subnet_n(ssn_engine* eng, uint32_t id, const ssn_subnet_cfg* cfg,
                          const float* bn_mean, const float* bn_var, uint64_t n_stats);

/* Build the LayerSelect CUDA-graph segments for every batch in the grid
 * (the catalog's profiled batch sizes, reference profile.hpp:164-171). */
int ssn_prepare(ssn_engine* eng, const uint32_t* batch_grid, uint32_t n);

/* Actuate subnet `id` in place: selects its plan; moves no weights. */
int ssn_actuate(ssn_engine* eng, uint32_t id);

/* Run the actuated subnet on `count` images padded to `profiled_batch`
 * (reference ClampedDispatch, policy.hpp:219-232).  `x` and `logits` may be
 * host or device pointers; logits are float32 [count][num_classes].
 * Enqueued on `stream` (cudaStream_t, NULL = engine stream); returns after
 * enqueue — call ssn_synchronize() before reading host logits.
 * Forwards of one engine share its arena, staged input and active-subnet
 * word: a forward enqueued on a different stream than the engine's previous
 * call is ordered after that call (an engine-owned event), so streams may be
 * mixed but forwards of one engine never overlap on the device. */
int ssn_forward(ssn_engine* eng, const void* x, uint32_t count,
                uint32_t profiled_batch, float* logits, void* stream);

int ssn_synchronize(ssn_engine* eng, void* stream);

/* Median device latency (CUDA events) of `iters` forwards of subnet `id` at
 * `batch` — the supernet profiler row l_phi(B) (reference profile.hpp:344). */
int ssn_profile_latency(ssn_engine* eng, uint32_t id, uint32_t batch,
                        uint32_t iters, double* median_us);

/* Per-op median device time (µs, CUDA events around each op, ops launched
 * back to back outside the graphs) of subnet `id` at `batch`; op_us has one
 * entry per supernet op (ssn_plan_ops order), 0 for skipped ops.  Feeds the
 * per-kernel roofline accounting. */
int ssn_profile_ops(ssn_engine* eng, uint32_t id, uint32_t batch,
                    uint32_t iters, float* op_us, uint32_t n_ops);

int ssn_query(ssn_engine* eng, ssn_stats* out);

/* Device pointer of the engine's last output logits (float32). */
int ssn_device_logits(ssn_engine* eng, const float** out);

/* Debugging: run subnet `id` op by op (no graphs) on the last staged input
 * and store an FNV-1a hash of every op's output in sums[op] (0 = not run). */
int ssn_debug_op_checksums(ssn_engine* eng, uint32_t id, uint32_t batch, uint64_t* sums,
                           uint32_t n_ops);
const char* ssn_last_error(void);

/* ---- operator-level entry points (the paper's operators on raw device
 * tensors).  All pointers are device pointers, NHWC. ---- */

/* WeightSlice conv + SubnetNorm + activation + residual, bf16 tcgen05 path.
 * x: [n][h][w][cin]  (compact, cin active channels, cin % 8 == 0)
 * wgt: max-shape KRSC [cout_max][k][k][cin_max] bf16, read as a leading
 *      slice [:cout][:, :][:cin] through a TMA tensor map (never copied)
 * scale/shift: float32 [cout] (NULL -> 1 / 0); res: [n][ho][wo][cout] or NULL
 * y: [n][ho][wo][cout] bf16, or float32 when out_f32 != 0
 * act: 0 none, 1 relu */
int ssn_op_conv_bf16(const void* x, int n, int h, int w, int cin,
                     const void* wgt, int cout_max, int cin_max, int k,
                     int stride, int pad, int cout, const float* scale,
                     const float* shift, const void* res, int act, int out_f32,
                     void* y, void* stream);

/* Depthwise WeightSlice conv (OFA elastic kernel) + SubnetNorm + activation,
 * bf16 (the OFA-MBv3 dw layers of ssn_forward run this kernel):
 * x: [n][h][w][c] bf16 compact (c % 8 == 0); y: [n][ho][wo][c] bf16
 * wgt: bf16 tap-major [k_max][k_max][c_max]; the active k x k kernel is the
 *      centre crop, the active channels the leading c (read in place)
 * pad = k / 2; scale/shift float32 [c] (NULL -> 1 / 0)
 * act: 0 none, 1 relu, 2 h_swish.  k in {3, 5, 7} <= k_max <= 7, stride 1/2.
 * Replaces the per-request worker sleep for these layers (serve_runtime.hpp:167). */
int ssn_op_dw_bf16(const void* x, int n, int h, int w, int c, const void* wgt,
                   int c_max, int k_max, int k, int stride, const float* scale,
                   const float* shift, int act, void* y, void* stream);

/* Same operator, float32 SIMT path (config-1 parity precision). groups ==
 * cin means depthwise with weights [c_max][k_max][k_max] centre-cropped to k. */
int ssn_op_conv_f32(const float* x, int n, int h, int w, int cin,
                    const float* wgt, int cout_max, int cin_max, int k_max,
                    int k, int stride, int pad, int cout, int depthwise,
                    const float* scale, const float* shift, const float* res,
                    int act, float* y, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SSN_H */
