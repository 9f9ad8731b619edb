/*
 * lane_b200.h -- C ABI of the B200-native FC-backprop hot path.
 *
 * This is the drop-in boundary for the reference's layer/network API
 * (/root/reference/proj/include/lane/{layers,network}.hpp).  The reference
 * reaches its backward kernels through lane::TaskSchedule / lane::KernelBody
 * (include/lane/task_runtime.hpp:24-42, :140-185): a per-index host closure
 * over host std::spans with per-execute copy-in/copy-out.  A CUDA kernel cannot
 * sit behind that interface, so the boundary is one level up:
 * the LayerState buffers and the layer/network methods that execute the
 * schedules.  Each entry point below names the reference interface it
 * replaces (file:line into /root/reference/proj).  The C++ facade in
 * include/lane_b200/lane.hpp restores the reference's class/exception API on
 * top of these functions; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *  - Every function returns an int status (LANE_OK == 0).  Non-zero codes
 *    mirror lane::Error's hierarchy (include/lane/error.hpp:8-38) plus CUDA and
 *    NCCL failures; lane_b200_last_error() returns the thread's last message.
 *    No C++ exception crosses the ABI.
 *  - Plain pointers and sizes only.  "host" pointers are ordinary CPU memory
 *    (pinned or pageable); "dev" pointers are device addresses on the
 *    context's GPU (e.g. from lane_b200_dev_alloc or torch tensors).
 *  - All state lives in HBM: weights, gradients, delta_weights, biases and the
 *    per-sample activation/delta buffers of every layer are device-resident for
 *    the life of the network -- no per-step host round trips (the reference's
 *    copy-in/copy-out, src/task_runtime.cpp:272-301, is gone).  Host copies
 *    happen only in *_host entry points, buf_read/buf_write and init.
 *  - Calls are stream-ordered on the context's stream; only functions that
 *    return host data (buf_read, *_stats outputs, sync) block.  One context per
 *    GPU, driven from one host thread (the reference's one-owner rule,
 *    include/lane/task_runtime.hpp:123-126).
 *  - fp32 everywhere (SPEC: fp32), weights row-major cols_input x cols_out
 *    ([i*out + o], include/lane/tensor.hpp:46-57).
 */
#ifndef LANE_B200_H
#define LANE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LANE_B200_ABI_VERSION 1

/* status codes: 1..6 mirror lane::ShapeError, ConfigError, ScheduleError,
 * TrainingError, IoError, ParseError (include/lane/error.hpp:12-38) */
enum {
    LANE_OK = 0,
    LANE_ERR_SHAPE = 1,
    LANE_ERR_CONFIG = 2,
    LANE_ERR_SCHEDULE = 3,
    LANE_ERR_TRAINING = 4,
    LANE_ERR_IO = 5,
    LANE_ERR_PARSE = 6,
    LANE_ERR_CUDA = 7,
    LANE_ERR_NCCL = 8,
    LANE_ERR_INTERNAL = 9
};

/* LayerState buffers, include/lane/layers.hpp:78-86 */
enum {
    LANE_BUF_W = 0,            /* weights        cols_input x cols_out */
    LANE_BUF_G = 1,            /* gradients      cols_input x cols_out */
    LANE_BUF_DW = 2,           /* delta_weights  cols_input x cols_out (momentum velocity) */
    LANE_BUF_B = 3,            /* biases         cols_out */
    LANE_BUF_INPUTS = 4,       /* inputs         cols_input   (row 0 of the batch) */
    LANE_BUF_NETIN = 5,        /* netin          cols_out     (row 0 of the batch) */
    LANE_BUF_OUTPUTS = 6,      /* outputs        cols_out     (row 0 of the batch) */
    LANE_BUF_DELTAS = 7,       /* deltas         cols_out     (row 0 of the batch) */
    LANE_BUF_DELTA_BIASES = 8, /* delta_biases   cols_out */
    LANE_BUF_BIAS_GRAD = 9,    /* extension: mean bias gradient (mini-batch) */
    LANE_BUF_COUNT = 10
};

/* Numerics mode.  STRICT reproduces the reference's evaluation order and
 * rounding (ascending sequential sums, no FMA contraction) so backward and
 * update results are bit-identical to the CPU reference given identical
 * inputs.  FAST uses split/tree reductions with FMA; results agree within the
 * condition-aware tolerance |gpu - cpu| <= 1e-5 * sum_k |a_k b_k|. */
enum { LANE_NUMERICS_STRICT = 0, LANE_NUMERICS_FAST = 1 };

typedef struct lane_b200_ctx lane_b200_ctx;
typedef struct lane_b200_net lane_b200_net;
typedef struct lane_b200_dataset lane_b200_dataset;

/* ----------------------------------------------------------- context --- */
int lane_b200_abi_version(void);
const char* lane_b200_last_error(void);
/* One context per GPU (replaces lane::Device, include/lane/task_runtime.hpp:97-127). */
int lane_b200_ctx_create(int device, lane_b200_ctx** out);
int lane_b200_ctx_destroy(lane_b200_ctx* ctx);
int lane_b200_ctx_set_numerics(lane_b200_ctx* ctx, int mode);
int lane_b200_ctx_get_numerics(lane_b200_ctx* ctx, int* mode);
/* Blocks until all work queued on the context's stream has finished. */
int lane_b200_sync(lane_b200_ctx* ctx);
/* The context's cudaStream_t, as an opaque pointer (for interop/timing). */
int lane_b200_ctx_stream(lane_b200_ctx* ctx, void** stream);
/* Number of this library's kernels launched on the context so far. */
int lane_b200_kernel_launches(lane_b200_ctx* ctx, uint64_t* count);
/* Device scratch owned by the context (freed with it).  */
int lane_b200_dev_alloc(lane_b200_ctx* ctx, size_t bytes, void** dev);
int lane_b200_dev_free(lane_b200_ctx* ctx, void* dev);
int lane_b200_memcpy_h2d(lane_b200_ctx* ctx, void* dev, const void* host, size_t bytes);
int lane_b200_memcpy_d2h(lane_b200_ctx* ctx, void* host, const void* dev, size_t bytes);

/* ----------------------------------------------------------- network --- */
/* FeedForwardNetwork(input_width, hidden_sizes, classes), network.hpp:14-30 /
 * network.cpp:25-45: all buffers zero.  max_batch sizes the activation
 * buffers for the mini-batch extension (>= 1). */
int lane_b200_net_create(lane_b200_ctx* ctx, size_t input_width, const size_t* hidden,
                         size_t n_hidden, size_t classes, size_t max_batch, lane_b200_net** out);
/* build_network's initialisation (network.cpp:55-66): weights of every layer,
 * hidden first then output, uniform in [-1/sqrt(fan_in), 1/sqrt(fan_in)) from
 * SplitMix64(seed) (tensor.hpp:13-44), biases zero -- bit-identical to the
 * reference; generated on the host once and uploaded. */
int lane_b200_net_init_seeded(lane_b200_net* net, uint64_t seed);
int lane_b200_net_destroy(lane_b200_net* net);
/* n_layers = n_hidden + 1; layer index n_hidden is the softmax output layer. */
int lane_b200_net_shape(lane_b200_net* net, size_t layer, size_t* cols_input, size_t* cols_out);
int lane_b200_net_n_layers(lane_b200_net* net, size_t* n_layers);
/* Host <-> device copies of one LayerState buffer (count = its element count). */
int lane_b200_buf_read(lane_b200_net* net, size_t layer, int buf, float* host, size_t count);
int lane_b200_buf_write(lane_b200_net* net, size_t layer, int buf, const float* host,
                        size_t count);
int lane_b200_buf_device_ptr(lane_b200_net* net, size_t layer, int buf, float** dev,
                             size_t* count);
/* FNV-1a over weights and biases, hidden then output (bench.cpp:32-41). */
int lane_b200_net_hash(lane_b200_net* net, uint64_t* hash);

/* ---------------------------------------------- layer API (B = 1) --- */
/* FullyConnectedLayer::forward / SoftmaxOutputLayer::forward
 * (layers.hpp:99,110; layers.cpp:27-49, :71-87).  x_host == NULL chains from
 * the previous layer's device outputs (layer > 0). */
int lane_b200_layer_forward(lane_b200_net* net, size_t layer, const float* x_host, size_t len);
/* FullyConnectedLayer::backward(next_weights, next_deltas, eta)
 * (layers.hpp:101-103, layers.cpp:51-69): fc_backward_tuple over (o, i).
 * next_W_host == NULL uses layer+1's device weights and deltas.  ShapeError
 * when next_W_rows != cols_out or next_d_len != next_W_cols. */
int lane_b200_fc_backward(lane_b200_net* net, size_t layer, const float* next_W_host,
                          size_t next_W_rows, size_t next_W_cols, const float* next_d_host,
                          size_t next_d_len, float eta);
/* SoftmaxOutputLayer::backward(target, eta) (layers.hpp:113, layers.cpp:89-102);
 * ShapeError when target_len != classes.  ConfigError when !(eta > 0)
 * (LearningRate, layers.hpp:11-19). */
int lane_b200_softmax_backward(lane_b200_net* net, const float* target_host, size_t target_len,
                               float eta);
/* LayerState::apply_updates (layers.hpp:75, layers.cpp:18-25): additive. */
int lane_b200_apply_updates(lane_b200_net* net, size_t layer);

/* ---------------------------------------------- network API (B = 1) --- */
/* FeedForwardNetwork::forward (network.cpp:47-53); probs_host may be NULL. */
int lane_b200_forward(lane_b200_net* net, const float* x_host, float* probs_host);
/* BackwardPlan::run (network.hpp:58-75, network.cpp:122-138): output backward,
 * hidden backward in reverse, then apply_updates on every layer; G and DW
 * are materialised exactly as the reference's stream_out leaves them. */
int lane_b200_backward_plan_run(lane_b200_net* net, const float* target_host, float eta);
/* The same step returning its std::vector<PhaseTiming> (network.hpp:70-72,
 * task_runtime.hpp:53-60): phase_ms[3*k + {0,1,2}] = copy_in, kernel,
 * copy_out milliseconds of schedule k, k = 0 the output layer then the hidden
 * layers in reverse (the order run() executes them); n_phase >= 3 * n_layers.
 * Times are CUDA events on the context's stream: copy_in is the target's
 * upload (output layer) and 0 for hidden layers, whose inputs are already
 * device-resident; copy_out is 0 (nothing leaves the device).  apply_updates
 * runs after the schedules, untimed, as in the reference.  Blocks. */
int lane_b200_backward_plan_run_timed(lane_b200_net* net, const float* target_host, float eta,
                                      double* phase_ms, size_t n_phase);

/* Fused online SGD over a device-resident sample stream: for s in [0, n_steps):
 * k = order[s] (order_dev == NULL => s mod n); FeedForwardNetwork::forward(X[k]);
 * cross_entropy/argmax (network.cpp:165-168); BackwardPlan::run(T[k]).  One
 * persistent kernel; weights stay on chip between samples.  Accumulates the
 * reference's loss_sum (double, sample order) and correct count into
 * *loss_sum_dev / *correct_dev (device; may be NULL).  After the call every
 * LayerState buffer holds what the reference leaves after the last sample
 * (G/DW of the last sample included).  X_dev: n x input_width, T_dev: n x
 * classes, row-major fp32. */
int lane_b200_sgd_stream(lane_b200_net* net, const float* X_dev, const float* T_dev, size_t n,
                         const uint32_t* order_dev, size_t n_steps, float eta,
                         double* loss_sum_dev, uint64_t* correct_dev);
/* Which fused plan lane_b200_sgd_stream runs for this network under the
 * context's current numerics/environment: writes a NUL-terminated description
 * ("window D=2 KS=2 ctas=65", "cluster ctas=16", "grid ...", or "layer" for the
 * per-sample layer-kernel path) into buf (len >= 64 recommended). */
int lane_b200_sgd_stream_plan(lane_b200_net* net, char* buf, size_t len);
/* train (network.hpp:77-82, network.cpp:140-182): per epoch the reference's
 * SplitMix64 Fisher-Yates shuffle (order not reset between epochs), one fused
 * sgd_stream over the epoch, EpochStats readback, early stop when
 * mean_loss <= max_error.  Inputs are host arrays (uploaded once).  Writes up
 * to max_epochs (mean_loss, accuracy) pairs; *epochs_run receives the count.
 * TrainingError for an empty set. */
int lane_b200_train(lane_b200_net* net, const float* X_host, const float* T_host, size_t n,
                    float eta, float max_error, size_t max_epochs, uint64_t seed,
                    float* mean_loss_out, float* accuracy_out, size_t* epochs_run);
/* evaluate (network.hpp:86, network.cpp:184-204). */
int lane_b200_evaluate(lane_b200_net* net, const float* X_host, const float* T_host, size_t n,
                       float* mean_loss, float* accuracy);

/* --------------------------------- mini-batch extension --- */
/* One step on a device-resident batch (B <= max_batch):
 *   G = (1/B) sum_b delta_b (x) x_b ;  DW = mu*DW + (-eta)*G (DW = -eta*G when
 *   mu == 0) ; W += DW ; same for the biases.  Every delta uses pre-update
 *   weights.  B == 1, mu == 0 reduces to BackwardPlan::run.  ConfigError
 *   unless eta > 0 and 0 <= mu < 1.  When the context has a communicator
 *   (lane_b200_comm_init) the gradient sums are all-reduced across ranks
 *   before the update (one NCCL fp32 allreduce per layer, issued right after
 *   that layer's wgrad so it overlaps the rest of the backward), and
 *   B_global = B * world.  loss_sum_dev (device double, may be NULL)
 *   accumulates the local cross entropy. */
int lane_b200_minibatch_step(lane_b200_net* net, const float* X_dev, const float* T_dev,
                             size_t B, float eta, float mu, double* loss_sum_dev);

/* The same step in its three data-parallel phases (the SURVEY 8b sketch's
 * lane_b200_backward / lane_b200_allreduce_grads / lane_b200_apply_updates(net,
 * momentum)); minibatch_step == grads, then the per-layer allreduce, then
 * apply(B * world), bit for bit.
 * minibatch_grads: forward + backward of a device batch (B <= max_batch);
 *   leaves the gradient SUMS over the B rows (sum_b delta_b (x) x_b and
 *   sum_b delta_b, not yet divided) in the grads arena; no update, no
 *   communication.  loss_sum_dev as in minibatch_step.
 * minibatch_apply: the update from the arena's (summed) gradients:
 *   G = gsum / B_global; DW = mu*DW + (-eta)*G; W += DW; biases alike; G and
 *   the bias gradients are left as the means.  ConfigError unless eta > 0 and
 *   0 <= mu < 1.  delta_weights is the velocity: whatever update was last
 *   applied to the layer (by a mini-batch step or by the online path's last
 *   sample, which leaves DW = -eta*G of that sample, as the reference does).
 * net_grads_arena: the flat gradient arena, [G_0 | gb_0 | G_1 | gb_1 | ...]
 *   (256-byte aligned pieces, zero padding), the buffer an allreduce sums. */
int lane_b200_minibatch_grads(lane_b200_net* net, const float* X_dev, const float* T_dev, size_t B,
                              double* loss_sum_dev);
int lane_b200_minibatch_apply(lane_b200_net* net, size_t B_global, float eta, float mu);
int lane_b200_net_grads_arena(lane_b200_net* net, float** dev, size_t* count);

/* Mini-batch training over a host dataset (the input side of the
 * path).  X_host [n][input_width], T_host [n][classes] (pageable or pinned).
 * Each epoch permutes the sample order with SplitMix64(seed) when shuffle != 0
 * (one generator for the whole run, continuing the previous epoch's order, as
 * train does, network.cpp:153-161), then runs n / (batch * world) steps of
 * lane_b200_minibatch_step; rank r of a communicator takes rows
 * [r*batch, (r+1)*batch) of every global batch.  With world == 1 and
 * drop_last == 0 a final short step takes the n % batch remaining rows.
 * Input pipeline: the rows of a step are gathered on the host into one of 3
 * page-locked slots and copied on a second stream while earlier steps run;
 * each step's running loss is read back asynchronously.  mean_loss_out
 * [epochs] (local samples) and step_loss_out [epochs * steps] (mean loss of
 * each step) may be NULL; steps_run = steps executed over all epochs. */
int lane_b200_train_minibatch(lane_b200_net* net, const float* X_host, const float* T_host, size_t n,
                              size_t batch, float eta, float mu, size_t epochs, uint64_t seed, int shuffle,
                              int drop_last, float* mean_loss_out, float* step_loss_out, size_t* steps_run);

/* Diagnostic: one GEMM of the mini-batch path on device buffers (row-major):
 * op 0 NN: C[M,N] = A[M,K] B[K,N];  op 1 NT: C = A[M,K] B[N,K]^T;
 * op 2 TN: C = A[K,M]^T B[K,N].  epilogue 0 store, 1 +bias[n], 2 +bias[n]
 * with C2 = tanh(C), 3 C = (1 - aux^2) * acc.  use_tc: 0 the SIMT kernel;
 * 1 the tcgen05 3xTF32 kernels where the shape is eligible; 2 the persistent
 * stream-K 3xTF32 kernel for every eligible shape; 3 the one-tile-per-CTA
 * 3xTF32 kernels only; 4 the tcgen05 3xF16 kernel (power-of-two row/column
 * operand scales, kind::f16 MMAs); 5 the mini-batch step's own choice (3xF16
 * for the tall long-K shapes, 3xTF32 otherwise; LANE_B200_TC_PREC overrides). */
int lane_b200_gemm(lane_b200_ctx* ctx, int op, int M, int N, int K, const float* A, const float* B,
                   float* C, float* C2, const float* bias, const float* aux, int epilogue, int use_tc);
/* The same with caller-supplied 3xF16 operand maxima (float bits of max |.|):
 * amax per row of op(A) (M), bmax per column of op(B) (N), as
 * lane_b200_absmax computes them; used when the call runs the 3xF16 kernel
 * (the mini-batch step computes them once per step, not per GEMM). */
int lane_b200_gemm_ex(lane_b200_ctx* ctx, int op, int M, int N, int K, const float* A, const float* B,
                      float* C, float* C2, const float* bias, const float* aux, int epilogue, int use_tc,
                      const unsigned* amax, const unsigned* bmax);
/* max |x| (as float bits) of every row and every column of a row-major
 * rows x cols device matrix (cols % 4 == 0), one pass. */
int lane_b200_absmax(lane_b200_ctx* ctx, const float* X, int rows, int cols, unsigned* row_max,
                     unsigned* col_max);

/* ---------------------------------------------- datasets --- */
/* DataSet (include/lane/dataset.hpp:16-23) held by the library in page-locked
 * host memory (plain memory when no GPU is present): X [n][features] then
 * T [n][classes], row-major -- pass the pointers from dataset_info straight
 * to lane_b200_train / _train_minibatch / _evaluate. */
int lane_b200_dataset_create(size_t features, size_t classes, size_t n, const float* X, const float* T,
                             lane_b200_dataset** out);
/* load_dataset (dataset.hpp:25-30, dataset.cpp:31-83): CSV, features then a
 * one-hot label per line; IoError when the file cannot be opened, ParseError
 * with the line number for a bad field count, a non-numeric field (parsed as
 * std::from_chars), a label field other than 0/1 or a label that is not
 * one-hot.  Empty lines are skipped. */
int lane_b200_dataset_load(const char* path, size_t features, size_t classes, lane_b200_dataset** out);
/* save_dataset (dataset.hpp:32-33, dataset.cpp:85-103): %.9g features. */
int lane_b200_dataset_save(const lane_b200_dataset* d, const char* path);
int lane_b200_dataset_info(const lane_b200_dataset* d, size_t* features, size_t* classes, size_t* n, float** X,
                           float** T, int* pinned);
/* split (dataset.hpp:35-37, dataset.cpp:105-124): ConfigError unless
 * 0 < train_fraction < 1. */
int lane_b200_dataset_split(const lane_b200_dataset* d, double train_fraction, uint64_t seed,
                            lane_b200_dataset** train, lane_b200_dataset** test);
/* enlarge (dataset.hpp:39-41, dataset.cpp:126-148); *rng_state is the
 * SeededRng state (tensor.hpp:13-44), advanced in place.  ConfigError for
 * factor == 0 or noise < 0. */
int lane_b200_dataset_enlarge(const lane_b200_dataset* d, size_t factor, float noise, uint64_t* rng_state,
                              lane_b200_dataset** out);
int lane_b200_dataset_destroy(lane_b200_dataset* d);

/* ------------------------------------------- multi-GPU (data parallel) --- */
int lane_b200_nccl_unique_id(void* id_out, size_t id_bytes); /* id_bytes >= 128 */
int lane_b200_comm_init(lane_b200_ctx* ctx, int rank, int world, const void* id,
                        size_t id_bytes);
int lane_b200_comm_destroy(lane_b200_ctx* ctx);
/* All-reduce (sum) the flat gradient buffer of the network (G and bias
 * gradients of every layer) over the context's communicator. */
int lane_b200_allreduce_grads(lane_b200_net* net);

/* NVLink SHARP: the gradient exchange fused with the update
 * (csrc/nvls.cuh).  Once a network is NVLS-bound, lane_b200_minibatch_step /
 * lane_b200_train_minibatch reduce the gradient sums through the NVSwitch
 * (multimem.ld_reduce) and broadcast the updated W / velocities / mean
 * gradients (multimem.st), each rank one slice, instead of an NCCL allreduce
 * followed by a full local update; B_global = rows per step x world.
 * Sequence: rank 0 _nvls_create (exports a POSIX fd; fd_out may be NULL for a
 * single rank); every rank _nvls_attach (ranks != 0 import rank 0's fd);
 * a host barrier; every rank _nvls_bind; a host barrier.  *out = 1 when the
 * device supports multicast objects. */
int lane_b200_nvls_supported(lane_b200_ctx* ctx, int* out);
int lane_b200_nvls_create(lane_b200_net* net, int world, int* fd_out);
int lane_b200_nvls_attach(lane_b200_net* net, int rank, int world, int fd);
int lane_b200_nvls_bind(lane_b200_net* net);
/* *multicast = 1 (bound to a multicast object), 0 (one rank, "local": the GPU
 * slice could not create a multicast object, so the same slice / update /
 * barrier kernels run with plain memory operations), -1 (not bound). */
int lane_b200_nvls_mode(lane_b200_net* net, int* multicast);

#ifdef __cplusplus
}
#endif

#endif /* LANE_B200_H */
