/*
 * dpb.h — C ABI of the B200-native memory-efficient dense block.
 *
 * This is the drop-in boundary for the reference's hot path (denseplan,
 * arXiv 1707.06990): the pre-activation bottleneck dense block
 *   cat -> BN_a -> ReLU -> conv1x1 -> BN_b -> ReLU -> conv3x3
 * forward and backward with shared storage and recompute-on-backward.
 * Plain C: pointers, sizes and status codes only; no C++ or torch types.
 *
 * Reference interfaces replaced (paths relative to /root/reference/proj):
 *   dpb_block_plan          GraphPlan<T>::build pool sizing + PoolRegion /
 *                           GradPool / BufferPool  include/denseplan/graph.hpp:28-127,
 *                           :456-482, :602-609 (one block's share)
 *   dpb_block_forward       GraphPlan<T>::forward layer loop over forward_layer
 *                           include/denseplan/graph.hpp:747-760, :618-670
 *   dpb_block_backward      GraphPlan<T>::backward_block -> backward_layer with
 *                           rematerialize   include/denseplan/graph.hpp:1054-1063,
 *                           :856-945, :831-854
 *   dpb_op_*                the per-op kernels of include/denseplan/ops.hpp
 *                           (batch_statistics :138-162, batchnorm_apply :115-134,
 *                           batchnorm_backward :206-243, conv2d_forward :315-342,
 *                           conv2d_backward :346-387)
 *   dpb_count_parameters,   densenet.hpp:234-275, peak_model.hpp:37-158
 *   dpb_predict_peak_elements
 *   status codes            errors.hpp:8-61 (1:1, declaration order)
 *
 * Conventions
 *   - Every entry point returns int status: 0 OK; 1..12 the reference error
 *     classes in declaration order; >= 100 CUDA / NCCL failures.
 *     dpb_last_error() returns a thread-local message for the last failure.
 *   - All tensor pointers passed to device entry points are DEVICE pointers
 *     owned by the caller; the block handle owns its HBM arena.  Calls are
 *     asynchronous on the handle's stream; dpb_sync() surfaces async errors.
 *   - Reference-facing tensors are fp32 NCHW (dp/tensor.hpp:102-108).  The
 *     block's internal layout is NHWC in the arena.
 *   - Flat per-block parameter layout (reference registration order,
 *     graph.hpp:459-478), layer l with c = c0 + l*k input channels:
 *         gamma_a[c] beta_a[c] W1[bk][c] gamma_b[bk] beta_b[bk] W2[k][bk][3][3]
 *     Gradients use the same layout.  Statistics / running statistics:
 *         mean_a[c] var_a[c] mean_b[bk] var_b[bk]       per layer.
 *   - One handle per GPU, used by one host thread at a time (the reference
 *     plan is single-threaded, alloctrace.hpp:55-56).
 */
#ifndef DPB_H_
#define DPB_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DPB_API __attribute__((visibility("default")))
#else
#define DPB_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: errors.hpp declaration order */
enum {
  DPB_OK = 0,
  DPB_SHAPE_ERROR = 1,
  DPB_BOUNDS_ERROR = 2,
  DPB_SIZE_OVERFLOW_ERROR = 3,
  DPB_CAPACITY_ERROR = 4,
  DPB_ACCOUNTING_ERROR = 5,
  DPB_CONFIG_ERROR = 6,
  DPB_FORMAT_ERROR = 7,
  DPB_LABEL_ERROR = 8,
  DPB_DEGENERATE_BATCH_ERROR = 9,
  DPB_PROTOCOL_ERROR = 10,
  DPB_RANGE_ERROR = 11,
  DPB_VERIFY_ERROR = 12,
  DPB_CUDA_ERROR = 100,
  DPB_NCCL_ERROR = 101
};

/* storage precision of features / bottleneck outputs inside the arena */
enum { DPB_FP32 = 0, DPB_BF16 = 1 };

/* layout of the reference-facing block input / gradient tensors */
enum { DPB_NCHW = 0, DPB_NHWC = 1 };

/* arena tags: alloctrace.hpp:17-24 */
enum {
  DPB_ARENA_PARAMS = 0,
  DPB_ARENA_FEATURE_OWNED = 1,
  DPB_ARENA_SHARED1 = 2,
  DPB_ARENA_SHARED2 = 3,
  DPB_ARENA_SHARED_GRAD = 4,
  DPB_ARENA_SCRATCH = 5
};

typedef struct dpb_block_desc {
  int64_t n, h, w; /* batch and spatial size inside the block */
  int32_t c0;      /* channels entering the block */
  int32_t m;       /* bottleneck layers */
  int32_t k;       /* growth rate */
  int32_t bk;      /* bottleneck width (4k in DenseNet-BC) */
  int32_t dtype;   /* DPB_FP32 (1e-4 parity path) or DPB_BF16 (tensor path) */
  int32_t layout;  /* DPB_NCHW or DPB_NHWC for x_in / grad_acc */
} dpb_block_desc;

/* Byte layout of one block's HBM arena (host-side plan, no allocation). */
typedef struct dpb_arena_sizes {
  int64_t total_bytes;
  /* persistent over fwd->bwd (FeatureOwned: the O(m) part) */
  int64_t feat_offset, feat_bytes;   /* [M, c_out] features (x_in | y_1..y_m)  */
  int64_t z_offset, z_bytes;         /* m x [M, bk] bottleneck outputs          */
  int64_t stats_offset, stats_bytes; /* per-channel batch mean/var               */
  /* SharedGrad: block accumulator + two transient slots */
  int64_t acc_offset, acc_bytes;     /* [M, c_out] fp32                          */
  int64_t g0_offset, g0_bytes;       /* [M, bk]   fp32 masked 3x3 dgrad          */
  int64_t g1_offset, g1_bytes;       /* 2 x [M, c_max] fp32 masked 1x1 dgrad (layer parity) */
  /* Scratch: reduction partials, GEMM-layout weight copies */
  int64_t scratch_offset, scratch_bytes;
  /* Shared1/Shared2 of the reference are 0: concat is a zero-copy channel
   * prefix and BN+ReLU are recomputed inside the conv prologues. */
  int64_t shared1_bytes, shared2_bytes;
  int64_t param_elems;   /* flat parameter count of the block             */
  int64_t stat_elems;    /* flat statistics count of the block            */
} dpb_arena_sizes;

typedef struct dpb_block dpb_block;

/* Device-memory accounting of a handle (MemoryStats, alloctrace.hpp:40-50):
 * live / peak bytes per arena tag (DPB_ARENA_*), the combined feature peak
 * (every arena but Params) and the parameter bytes.  libdpb records every
 * device allocation it makes, split by the regions it holds:
 * FeatureOwned = features, bottleneck outputs, batch statistics (and, for a
 * model, the stem / transition activations); SharedGrad = the block
 * accumulators and the gradient transients; Scratch = reduction partials and
 * the pre-tiled bf16 weight images.  Shared1 / Shared2 stay 0 (concat and
 * BN+ReLU are recomputed inside the conv prologues).  Parameters and
 * gradients are caller-owned and not counted. */
typedef struct dpb_memory_stats {
  int64_t live_bytes[6];
  int64_t peak_bytes[6];
  int64_t total_feature_peak_bytes;
  int64_t param_bytes;
} dpb_memory_stats;

DPB_API const char* dpb_last_error(void);
DPB_API const char* dpb_version(void);

/* Host-only: validate the descriptor and compute the arena layout. */
DPB_API int dpb_block_plan(const dpb_block_desc* desc, dpb_arena_sizes* out);
DPB_API int dpb_block_param_elems(const dpb_block_desc* desc, int64_t* param_elems,
                          int64_t* stat_elems);

/* Allocate the arena on `device`; `stream` is a cudaStream_t (NULL = legacy
 * default stream). */
DPB_API int dpb_block_create(const dpb_block_desc* desc, int device, void* stream,
                     dpb_block** out);
DPB_API int dpb_block_destroy(dpb_block* blk);
DPB_API int dpb_block_set_stream(dpb_block* blk, void* stream);
DPB_API int dpb_block_arena(dpb_block* blk, dpb_arena_sizes* out, void** base);

/* Forward (train mode).  x_in: [n, c0, h, w] fp32 (or NHWC per desc).
 * params: flat fp32 device array.  running: flat fp32 running stats, updated
 * in place with momentum 0.1 / biased variance when update_running != 0
 * (ops.hpp:185-194).  After the call the arena holds the block output
 * features, the bottleneck outputs and the batch statistics.  DegenerateBatch
 * (9) when n*h*w < 2. */
DPB_API int dpb_block_forward(dpb_block* blk, const float* x_in, const float* params,
                      float* running, int update_running);

/* Eval mode: normalise with the running statistics (ops.hpp:196-199). */
DPB_API int dpb_block_forward_eval(dpb_block* blk, const float* x_in,
                           const float* params, const float* running);

/* Backward.  grad_acc: [n, c_out, h, w] fp32 gradient w.r.t. the block output
 * (as written by the consumer's BN backward, graph.hpp:1117-1120); on return
 * it holds the full block-gradient accumulator, whose prefix [0, c0) is the
 * gradient w.r.t. the block input (graph.hpp:1138, :1172-1173).  grads: flat
 * fp32, written (not accumulated) like conv2d_backward / batchnorm_backward.
 * Protocol error (10) if no train-mode forward preceded it. */
DPB_API int dpb_block_backward(dpb_block* blk, const float* params, float* grad_acc,
                       float* grads);

/* Read back arena contents in the reference's NCHW fp32 layout. */
DPB_API int dpb_block_read_feats(dpb_block* blk, float* dst /* [n, c_out, h, w] */);
DPB_API int dpb_block_read_z(dpb_block* blk, float* dst /* m x [n, bk, h, w] */);
DPB_API int dpb_block_read_stats(dpb_block* blk, float* dst /* flat stats layout */);

DPB_API int dpb_sync(dpb_block* blk);
DPB_API int dpb_block_memory_stats(dpb_block* blk, dpb_memory_stats* out);
/* OpTrace of the last forward + backward (alloctrace.hpp:132-201, FLOP
 * conventions ops.hpp:565-595): counts[3 * node + {0 forward, 1 backward,
 * 2 recompute}] for nodes 7l + {concat, bn_a, relu_a, conv_a, bn_b, relu_b,
 * conv_b} and 7m (block-output concat); flops[7 * {0,1,2} + OpKind] with
 * OpKind concat 0, batchnorm 1, relu 2, conv 3.  The concat is a zero-copy
 * view (no moves, 0 FLOPs); act_a and act_b are recomputed twice per layer
 * (dgrad mask and wgrad operand), inside the kernels' prologues. */
DPB_API int dpb_block_trace(dpb_block* blk, int32_t* counts, int max_nodes, double* flops, int* nodes);

/* Number of kernels the last forward/backward launched (bench accounting). */
DPB_API int64_t dpb_block_launch_count(dpb_block* blk);

/* Optional per-launch profiler: when enabled every kernel launch is bracketed
 * by CUDA events on the block's stream and tagged with its algorithmic HBM
 * bytes and FLOPs.  Enabling resets the record; reading
 * synchronises the stream and returns one entry per kernel category. */
typedef struct dpb_kernel_stat {
  char name[32];
  int64_t launches;
  double total_ms;
  double bytes;  /* algorithmic bytes summed over the launches (fp32 storage) */
  double flops;  /* algorithmic flops summed over the launches */
  double bytes_8d; /* the same under SURVEY 8(d)'s model: 2-byte activations, fp32 gradients */
} dpb_kernel_stat;
DPB_API int dpb_block_profile(dpb_block* blk, int enable);
DPB_API int dpb_block_profile_read(dpb_block* blk, dpb_kernel_stat* out, int max, int* count);
/* Peak device bytes the block's arena holds (efficient variant) and what a
 * naive store-everything variant of the same block would hold. */
DPB_API int dpb_block_memory(const dpb_block_desc* desc, int64_t* efficient_bytes,
                     int64_t* naive_bytes);

/* Diagnostic: D[M,N] = A . B^T on the tcgen05 engine with fp32 global
 * operands (A [M][K] or [K][M] when a_mn; B [N][K] or [K][N] when b_mn),
 * bf16 (split=0) or bf16x3 hi/lo (split=1) products, N tile bn in
 * {16,48,64,128,192}; colsum [ceil(M/128)][N][2] per-CTA column sums. */
DPB_API int dpb_selftest_tc_gemm(const float* A, const float* B, float* D, float* colsum,
                                 int M, int N, int K, int bn, int a_mn, int b_mn, int split,
                                 void* stream);

/* ---- per-op entry points (ops.hpp parity), fp32 NCHW device tensors ---- */
DPB_API int dpb_op_batch_statistics(const float* x, int64_t n, int64_t c, int64_t h,
                            int64_t w, float* mean, float* var, void* stream);
DPB_API int dpb_op_batchnorm_apply(const float* x, int64_t n, int64_t c, int64_t h,
                           int64_t w, const float* gamma, const float* beta,
                           const float* mean, const float* var, int relu,
                           float* dst, void* stream);
DPB_API int dpb_op_batchnorm_backward(const float* grad_y, const float* x, int64_t n,
                              int64_t c, int64_t h, int64_t w,
                              const float* gamma, const float* mean,
                              const float* var, float* grad_x,
                              float* grad_gamma, float* grad_beta,
                              void* stream);
DPB_API int dpb_op_conv2d_forward(const float* x, int64_t n, int64_t cin, int64_t h,
                          int64_t w, const float* weights, int64_t cout,
                          int64_t kernel, int64_t pad, float* dst,
                          void* stream);
DPB_API int dpb_op_conv2d_backward(const float* grad_y, const float* x, int64_t n,
                           int64_t cin, int64_t h, int64_t w,
                           const float* weights, int64_t cout, int64_t kernel,
                           int64_t pad, float* grad_x /* may be NULL */,
                           float* grad_w, void* stream);

/* concat_forward / concat_backward (ops.hpp:53-107): input i (NCHW [n, c_i,
 * h, w]) <-> channels [sum_{j<i} c_j, ... + c_i) of the NCHW [n, c, h, w]
 * whole; strided device copies.  ShapeError for zero inputs, CapacityError
 * (forward) / ShapeError (backward) when the channels do not sum to c. */
DPB_API int dpb_op_concat_forward(int count, const float* const* inputs, const int64_t* channels, int64_t n,
                                  int64_t h, int64_t w, float* dst, int64_t dst_c, void* stream);
DPB_API int dpb_op_concat_backward(const float* grad_out, int64_t n, int64_t c, int64_t h, int64_t w, int count,
                                   const int64_t* channels, float* const* grads, void* stream);
/* relu_forward / relu_inplace (dst == x) and relu_backward(_inplace)
 * (ops.hpp:248-287): dst = x > 0 ? x : 0; grad_x = ref > 0 ? grad_y : 0. */
DPB_API int dpb_op_relu_forward(const float* x, int64_t count, float* dst, void* stream);
DPB_API int dpb_op_relu_backward(const float* grad_y, const float* ref, int64_t count, float* grad_x,
                                 void* stream);

/* ---- host-side model arithmetic (densenet.hpp / peak_model.hpp) -------- */
DPB_API int dpb_count_parameters(int nblocks, const int32_t* blocks, int32_t k,
                         int32_t bottleneck, double compression,
                         int32_t classes, int32_t c0, int32_t in_c,
                         int64_t* out);
/* strategy: 0 naive, 1 shared-gradient, 2 shared-all; out[6] per arena */
DPB_API int dpb_predict_peak_elements(int nblocks, const int32_t* blocks, int32_t k,
                              int32_t bottleneck, double compression,
                              int32_t classes, int32_t c0, int32_t strategy,
                              int64_t batch, int32_t in_c, int32_t in_h,
                              int32_t in_w, int64_t* out);

/* Rng(seed).normal() x count in the reference's draw order (rng.hpp:36-49) */
DPB_API int dpb_rng_fill_normal(uint64_t seed, float* host_dst, int64_t count);

/* ---- whole-network training step ----------------------
 * Replaces GraphPlan<T>::forward + compute_loss + backward
 * (graph.hpp:731-809, :811-826, :1065-1183) for the CIFAR-type network:
 *   stem conv3x3 -> [dense block -> transition (BN-ReLU-1x1 conv-2x2 avgpool)]*
 *   -> dense block -> head (BN-ReLU-global avgpool-linear) -> softmax-xent.
 * Dense blocks run through dpb_block_* (NHWC arenas); the transition computes
 * avgpool before its 1x1 conv (the two commute), on a quarter of the pixels.
 * Parameters and gradients: one flat fp32 buffer in the reference's
 * registration order (graph.hpp:356-390, :456-600):
 *   stem.w[c0][in_c][3][3] (stem 1: stem.conv.w[c0][in_c][7][7]
 *   stem.bn.gamma[c0] stem.bn.beta[c0]); per block its dpb_block layout; per transition
 *   bn.gamma[C] bn.beta[C] conv.w[c_out][C]; head.bn.gamma[C] head.bn.beta[C]
 *   head.linear.w[classes][C] head.linear.b[classes].
 * Running statistics in network order: (stem 1: stem.bn mean[c0] var[c0]), block 0 (its dpb_block layout),
 * transition 0 mean[C] var[C], block 1, ..., last block, head mean[C] var[C].
 * Bottleneck networks only. */
typedef struct dpb_model dpb_model;
typedef struct dpb_model_desc {
  int32_t nblocks;      /* 1..8 */
  int32_t blocks[8];    /* layers per block */
  int32_t k;            /* growth rate; bottleneck width 4k */
  double compression;   /* transition theta in (0, 1] */
  int32_t classes;
  int32_t c0;           /* stem output channels */
  int32_t in_c, in_h, in_w;
  int64_t batch;
  int32_t dtype;        /* DPB_FP32 | DPB_BF16 (dense blocks) */
  int32_t stem;         /* 0: the reference's conv 3x3/1 stem (graph.hpp:430, :740-745);
                           1: ImageNet stem conv 7x7/2 pad 3 -> BN -> ReLU -> max-pool
                           3x3/2 pad 1 (extension; 224 -> 112 -> 56) */
} dpb_model_desc;

DPB_API int dpb_model_sizes(const dpb_model_desc* desc, int64_t* param_elems, int64_t* running_elems);
/* GraphPlan<T>::build's parameter initialisation replayed draw for draw from
 * Rng(seed) (graph.hpp:351-390, :405-600; rng.hpp:36-49) into a HOST buffer of
 * dpb_model_sizes' param_elems floats: He-normal convs, BN gamma 1 / beta 0,
 * classifier N(0, 1/C), bias 0 — bit-identical to the reference's params()
 * for stem 0. */
DPB_API int dpb_model_init_params(const dpb_model_desc* desc, uint64_t seed, float* host_params);
DPB_API int dpb_model_create(const dpb_model_desc* desc, int device, void* stream, dpb_model** out);
DPB_API void dpb_model_destroy(dpb_model* model);
/* One training step: input NCHW [batch, in_c, in_h, in_w], labels int32
 * [batch] (device); writes grads (flat, registration order), updates running
 * statistics (momentum 0.1) and writes the mean loss to *loss (device float).
 * On a created stream that is not being captured, the first call captures the
 * step's launches into a CUDA graph and later calls with the same six buffers
 * replay it (DPB_MODEL_NO_GRAPH=1: always launch eagerly). */
DPB_API int dpb_model_step(dpb_model* model, const float* input, const int32_t* labels,
                           const float* params, float* running, float* grads, float* loss);
/* Waits for the step and surfaces its asynchronous errors: LabelError (8)
 * when a label was outside [0, classes) — that sample's loss and gradients
 * are NaN.  Gradients must not be used before dpb_model_sync succeeded. */
DPB_API int dpb_model_sync(dpb_model* model);
/* Makes `stream` (a cudaStream_t) wait until the last enqueued step has read
 * its input images and labels (the tensor-core stem: after the forward's loss;
 * otherwise after the step), so the next batch can be copied into the same
 * buffers while that step's backward still runs. */
DPB_API int dpb_model_wait_input(dpb_model* model, void* stream);
/* The model's device-memory accounting (every block arena + the stem,
 * transition and head buffers) and the number of kernels one training step
 * launches (the CUDA graph's kernel nodes once captured). */
DPB_API int dpb_model_memory_stats(dpb_model* model, dpb_memory_stats* out);
DPB_API int64_t dpb_model_launch_count(dpb_model* model);

/* ---- data parallelism ---------------------------------------------
 * One NCCL communicator per GPU, one process per GPU.  Rank 0 creates the id
 * (dpb_comm_unique_id, 128 bytes) and the caller distributes it (e.g. a
 * torch.distributed broadcast); every rank then calls dpb_comm_init.  With a
 * communicator attached (dpb_model_set_comm), dpb_model_step averages the
 * parameter gradients over the ranks (ncclAvg, fp32): one allreduce per
 * bucket, issued on the model's communication stream as soon as the bucket's
 * gradients exist (block b's parameters with its transition / the head,
 * right after block b's backward; the stem with block 0), overlapping the
 * backward of the blocks below, and joined before the step ends — inside the
 * step's CUDA graph.  BN statistics stay per rank.
 * dpb_model_buckets lists the buckets [begin, end) (flat parameter offsets)
 * in issue order; they tile [0, param_elems).  NCCL is loaded at run time
 * (the copy already in the process when there is one). */
typedef struct dpb_comm dpb_comm;
DPB_API int dpb_comm_unique_id(uint8_t* out /* 128 bytes */);
DPB_API int dpb_comm_init(int nranks, int rank, const uint8_t* id, int device, dpb_comm** out);
DPB_API int dpb_comm_destroy(dpb_comm* comm);
DPB_API int dpb_comm_check(dpb_comm* comm);  /* ncclCommGetAsyncError */
DPB_API int dpb_model_set_comm(dpb_model* model, dpb_comm* comm /* NULL: no exchange */);
DPB_API int dpb_model_buckets(const dpb_model_desc* desc, int64_t* ranges /* 2 * max */, int max, int* count);

/* ---- optimizer -------------------------------------------
 * dpb_sgd_step replaces sgd_step (train.hpp:43-70) over a flat fp32 buffer:
 *   d = g + wd*p;  v = mu*v + d;  p -= lr * (nesterov ? d + mu*v : v)
 * bit-identical to the reference's float loop; device pointers, async on
 * `stream`.  dpb_lr_at replaces lr_at (schedule.hpp:46-62): kind 0 = step
 * (milestones, factor), 1 = cosine (floor); RangeError outside [0, epochs). */
DPB_API int dpb_sgd_step(float* params, const float* grads, float* velocity, int64_t n, double lr,
                         double momentum, double weight_decay, int nesterov, void* stream);
DPB_API int dpb_lr_at(int kind, double base_lr, int total_epochs, const int32_t* milestones,
                      int nmilestones, double factor, double floor_lr, int epoch, double* out);

/* ---- DPLN checkpoints ---------------------------------------
 * save_checkpoint / load_checkpoint (checkpoint.hpp:121-198), fp32: `count`
 * entries with NUL-terminated names, dims[4*i .. 4*i+3] = (n, c, h, w) and
 * their elements concatenated in `data` (HOST memory).  Training checkpoints
 * (train.hpp:149-172) are the parameters in registration order followed by
 * "velocity.<name>" for each.  Load validates magic, version, element size,
 * count, names, shapes and the CRC-32 (FormatError otherwise). */
DPB_API int dpb_checkpoint_save(const char* path, int count, const char* const* names, const int64_t* dims,
                                const float* data, int epoch);
DPB_API int dpb_checkpoint_load(const char* path, int count, const char* const* names, const int64_t* dims,
                                float* data, int* epoch);

#ifdef __cplusplus
}
#endif

#endif /* DPB_H_ */
