/*
 * salt.h — C ABI of libsalt.so, the B200 (sm_100a) evaluator for fused
 * BLAS-1 expression trees (the hot path of SALT, arXiv 1109.1264).
 *
 * The reference (`lanevec`, pure Python + NumPy) has no native boundary:
 * its hot path is the pair of engine entry points
 *
 *     execute_assign(root, plan=None, *, backend, unroll, packages, stepped)
 *         pkg/src/lanevec/engine.py:295-311  -> _run_block_assign :243-264
 *     execute_reduce(root, plan=None, *, backend, unroll, packages, stepped)
 *         pkg/src/lanevec/engine.py:314-329  -> _run_block_reduce :267-292
 *
 * This header is the boundary that replaces those loops.  The Python host
 * layer (paper_1109_1264_b200/engine.py) keeps the reference signatures,
 * performs every validation the reference performs (and raises the same
 * exceptions) BEFORE calling in here, lowers the tree to a postfix
 * signature and calls one of the functions below through ctypes.
 *
 * Conventions
 *  - POD arguments only; no torch types.  Device pointers are BORROWED
 *    (never freed).  Element counts are int64 (config 5 has 2^31 elements).
 *  - `sig` is the canonical postfix tree signature, tokens separated by one
 *    space:  L<k> leaf k, S<k> scalar k, D (the value just assigned, only in
 *    the reduce tree of salt_assign_reduce), and the binary operators
 *    + - * (left operand first).  Examples:
 *        axpy  y + a*x              "L0 S0 L1 * +"        (L0 = y = dst)
 *        d = a + (b - c)            "L0 L1 L2 - +"
 *        d = al*a + be*(b - c)      "S0 L0 * S1 L1 L2 - * +"
 *        dot(x, y)                  "L0 L1 *"
 *  - scalars are passed as doubles that already hold the element-typed
 *    value (the Python side coerces them first, expressions.py:282).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).
 *  - Every function returns 0 on success and a negative SALT_E* code on
 *    failure; salt_last_error() returns a thread-local message.
 *  - Re-entrant: mutable state is limited to a once-initialised kernel
 *    table (mutex protected), per-device attribute caches and a
 *    thread-local error string.  Reduction scratch is caller-owned.
 */
#ifndef SALT_H
#define SALT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SALT_ABI_VERSION 1

/* per-tree limits of one fused kernel (larger trees are split by the host
 * layer into several fused evaluations through device temporaries) */
#define SALT_MAX_LEAVES  16
#define SALT_MAX_SCALARS 32

/* element types (lanes.py:31-43 accepts exactly f32 / f64) */
#define SALT_F32 0
#define SALT_F64 1

/* reduction flags */
#define SALT_SQRT    1 /* finish with sqrt in the element type (ops.norm2, ops.py:53-55) */
#define SALT_PARTIAL 2 /* write the per-device double-double partial {hi, lo} instead of
                          the rounded scalar (multi-GPU: all-gather then salt_reduce_finish) */

/* error codes */
#define SALT_OK          0
#define SALT_EINVAL     -1 /* bad signature / argument */
#define SALT_ECUDA      -2 /* CUDA runtime or driver failure */
#define SALT_EJIT       -3 /* NVRTC unavailable or compile failure */
#define SALT_EWORKSPACE -4 /* reduction workspace too small */

/* Elementwise assignment dst[i] = tree(leaves[.][i], scalars), i in [0, n).
 * Replaces engine.execute_assign (engine.py:295-311): one fused kernel, no
 * intermediate vector (AssignNode.block_commit, expressions.py:392-395).
 * dst may be identical to one of the leaves (exact aliasing, expressions.py
 * :326-333); shifted overlap is unsupported, as in the reference. */
int salt_assign(int dtype, const char* sig, void* dst,
                const void* const* leaves, int nleaves,
                const double* scalars, int nscalars,
                int64_t n, void* stream);

/* Reduction sum_i tree(leaves[.][i], scalars).  Replaces
 * engine.execute_reduce (engine.py:314-329) + SumNode.block_accumulate /
 * combine_partials (expressions.py:457-480).  Deterministic: fixed grid,
 * compensated (double-double) per-CTA partials combined in fixed order by
 * the last CTA.  out_dev receives one element of `dtype` (or, with
 * SALT_PARTIAL, one {double hi, double lo} pair).  If out_host is non-NULL
 * the result is also copied there and the stream is synchronised.
 * workspace must be >= salt_reduce_workspace_bytes() bytes of device memory,
 * zero-filled once before first use, and not shared by concurrent calls. */
int salt_reduce(int dtype, const char* sig,
                const void* const* leaves, int nleaves,
                const double* scalars, int nscalars,
                int64_t n, int flags,
                void* workspace, size_t workspace_bytes,
                void* out_dev, void* out_host, void* stream);

/* Fused assignment + reduction in ONE pass (BASELINE config 5, axpy -> dot):
 * dst[i] = assign_sig(...);  result = sum_i reduce_sig(..., D = dst[i]).
 * Replaces ops.axpy (ops.py:32-36) followed by ops.dot (ops.py:18-20),
 * which the reference runs as two traversals. */
int salt_assign_reduce(int dtype, const char* assign_sig, const char* reduce_sig,
                       void* dst, const void* const* leaves, int nleaves,
                       const double* scalars, int nscalars,
                       int64_t n, int flags,
                       void* workspace, size_t workspace_bytes,
                       void* out_dev, void* out_host, void* stream);

/* Several statements in ONE pass: up to SALT_MAX_ROOTS assignment roots
 * (postfix trees separated by ';' in assign_sigs; root r may read the value
 * root r' < r has just assigned as D<r'>) and optionally one reduction
 * (reduce_sig, may read D<r>; NULL for none).  Per element the roots run in
 * order, so the result equals running the statements one after another,
 * e.g. a conjugate-gradient update
 *     x = x + a*p ; r = r - a*q ; rr = sum(r*r)
 *     "L0 S0 L1 * + ; L2 S1 L3 * -"  with  "D1 D1 *",  dsts {x, r}.
 * assign_sigs may be NULL (a pure reduction).  Trees may also read up to
 * SALT_MAX_PSCALARS scalars from DEVICE memory as P<k> (pscalars[k] points
 * to one element of `dtype`): a solver's alpha computed on the GPU is used
 * without a host round trip, so whole iterations can be graph-captured. */
#define SALT_MAX_PSCALARS 8
#define SALT_MAX_ROOTS 4
int salt_fused(int dtype, const char* assign_sigs, const char* reduce_sig,
               void* const* dsts, int ndst, const void* const* leaves, int nleaves,
               const double* scalars, int nscalars,
               const void* const* pscalars, int npscalars,
               int64_t n, int flags,
               void* workspace, size_t workspace_bytes,
               void* out_dev, void* out_host, void* stream);

/* salt_fused with a SCALAR PROGRAM: the tree's device scalars P<k> are
 * computed once per thread in the kernel prologue from the raw device
 * scalars (pscalars[i], token "p<i>") and host scalars (scalars[j], "S<j>")
 * by a postfix program of "+ - * /" and "neg"; "=<k>" pops into P<k>.  E.g.
 * a CG step length alpha = rr / pq feeding x += alpha*p, r -= alpha*q:
 * scalar_prog "p0 p1 / =0" with pscalars {&rr, &pq} — one launch instead
 * of a division kernel plus the update.  Each op is one IEEE op in dtype
 * (the bits of the same arithmetic on 1-element device tensors).  At most
 * 32 ops, stack depth 8, 8 raw and 8 derived scalars; every P<k> the tree
 * reads must be written.  NULL / "" scalar_prog = salt_fused. */
int salt_fused_prog(int dtype, const char* assign_sigs, const char* reduce_sig,
                    void* const* dsts, int ndst, const void* const* leaves, int nleaves,
                    const double* scalars, int nscalars, const void* const* pscalars,
                    int npscalars, const char* scalar_prog, int64_t n, int flags,
                    void* workspace, size_t workspace_bytes, void* out_dev, void* out_host,
                    void* stream);

/* Combine `count` {hi, lo} partials (e.g. all-gathered from the ranks, in
 * rank order) in fixed order, round to dtype, optional SALT_SQRT. */
int salt_reduce_finish(int dtype, const void* partials_dev, int count, int flags,
                       void* out_dev, void* out_host, void* stream);

/* ---- sharded reductions: cross-GPU exchange over NVLink peer memory ----
 * Each rank owns a SALT_XCHG_BUFFER_BYTES symmetric device buffer (e.g. from
 * torch symmetric memory), zeroed once: 2 x 8 double-double slots followed
 * by 8 uint64 flags.  slots[p] / flags[p] are rank p's buffer (slot array /
 * flag array) mapped into this process.  epoch starts at 1 and increases by
 * one per exchange, identically on every rank.  The reduction kernel's last
 * CTA publishes this rank's total to every peer, waits for all of them and
 * folds them in rank order — the collective runs inside the reduction
 * kernel, with no NCCL call.  On timeout the result is NaN, *error = 1 and
 * the rank stores ABORT (~0) into its flag at every peer, which makes the
 * peers give up at once too; a rank whose *error is already set touches no
 * slot and aborts immediately (the error word is sticky: recreate the
 * buffers to recover).  Callers must check *error when a result is NaN. */
#define SALT_XCHG_MAX_RANKS 8
#define SALT_XCHG_BUFFER_BYTES 512
typedef struct salt_exchange {
  int32_t rank, world;
  uint64_t epoch;
  void* slots[SALT_XCHG_MAX_RANKS];
  void* flags[SALT_XCHG_MAX_RANKS];
  uint64_t timeout_ns; /* 0 = wait forever */
  void* error;         /* optional device uint32 */
} salt_exchange;

int salt_reduce_exchange(int dtype, const char* sig,
                         const void* const* leaves, int nleaves,
                         const double* scalars, int nscalars,
                         int64_t n, int flags,
                         void* workspace, size_t workspace_bytes,
                         const salt_exchange* exchange,
                         void* out_dev, void* out_host, void* stream);

int salt_assign_reduce_exchange(int dtype, const char* assign_sig, const char* reduce_sig,
                                void* dst, const void* const* leaves, int nleaves,
                                const double* scalars, int nscalars,
                                int64_t n, int flags,
                                void* workspace, size_t workspace_bytes,
                                const salt_exchange* exchange,
                                void* out_dev, void* out_host, void* stream);

/* salt_fused with the reduction's total exchanged in-kernel over NVLink
 * (as salt_reduce_exchange): statements + device scalars on sharded data.
 * reduce_sig must be non-NULL. */
int salt_fused_exchange(int dtype, const char* assign_sigs, const char* reduce_sig,
                        void* const* dsts, int ndst, const void* const* leaves, int nleaves,
                        const double* scalars, int nscalars,
                        const void* const* pscalars, int npscalars,
                        int64_t n, int flags,
                        void* workspace, size_t workspace_bytes,
                        const salt_exchange* exchange,
                        void* out_dev, void* out_host, void* stream);
int salt_fused_exchange_prog(int dtype, const char* assign_sigs, const char* reduce_sig,
                             void* const* dsts, int ndst, const void* const* leaves, int nleaves,
                             const double* scalars, int nscalars, const void* const* pscalars,
                             int npscalars, const char* scalar_prog, int64_t n, int flags,
                             void* workspace, size_t workspace_bytes, const salt_exchange* exchange,
                             void* out_dev, void* out_host, void* stream);

/* Test hook: `world` thread blocks of ONE cooperative launch play the ranks
 * of the exchange protocol for `rounds` consecutive epochs (epoch0 ...),
 * each block publishing totals[r*world + rank] ({hi, lo} pairs) and writing
 * the folded result to results[r*world + rank].  scratch: zeroed device
 * memory of world * SALT_XCHG_BUFFER_BYTES bytes. */
int salt_exchange_emulate(int world, int rounds, uint64_t epoch0,
                          const void* totals_dev, void* results_dev,
                          void* scratch_dev, void* stream);

/* ---- single-process multi-GPU: one host thread drives G devices ----
 * each device's reduction writes its {hi, lo} partial
 * (salt_reduce / salt_assign_reduce / salt_fused with SALT_PARTIAL); one
 * NCCL group of all-gathers over NVLink and a fixed rank-order fold leave
 * the total, rounded to dtype (sqrt with SALT_SQRT), in out_dev_per_gpu[g]
 * on every device — the bits of salt_reduce_finish / the in-kernel
 * exchange.  Replaces the reference's single-threaded Sum over the whole
 * vector (SumNode, expressions.py:401-480; engine.py:267-292) when the
 * vector is block-sharded across the devices of one process.
 *   out_dev_per_gpu[g]  device pointer on comms[g]'s device, >= 16 bytes:
 *                       the partial in, the scalar out (stream-ordered)
 *   comms               ncclComm_t[G] with comms[g] = rank g (e.g. from
 *                       salt_nccl_comm_init_all)
 *   streams             cudaStream_t[G], streams[g] on comms[g]'s device
 * Enqueues only (no host synchronisation).  NCCL is loaded at run time
 * ($SALT_NCCL_LIB, else libnccl.so.2). */
int salt_allreduce_sum(void* out_dev_per_gpu[], int G, int dtype, void* comms, void* streams[]);
int salt_allreduce_sum_flags(void* out_dev_per_gpu[], int G, int dtype, void* comms,
                             void* streams[], int flags);
/* ncclCommInitAll(G, devices) through the same runtime-loaded NCCL; comms_out
 * receives G ncclComm_t.  devices NULL = 0..G-1. */
int salt_nccl_comm_init_all(int G, const int* devices, void** comms_out);
int salt_nccl_comm_destroy(int G, void** comms);

/* Concurrent issue on the devices of one process (single-process multi-GPU,
 * devicegroup.py).  A group keeps one persistent host thread per member
 * device; salt_group_fused hands every member its own salt_fused call at
 * the same moment, so device g does not start g launch costs after device 0
 * (the serial issue loop the reference-side FFI would otherwise run).
 * Arguments are salt_fused's with per-member arrays (member-major):
 *   dsts      G x ndst        leaves    G x nleaves    pscalars G x npscalars
 *   ns[G]     lengths         ws[G]     workspaces (reduce modes)
 *   out_dev[G] results / SALT_PARTIAL partials     streams[G] per member
 * scalars are shared.  Enqueues only; returns after every member issued,
 * with the first failing member's code and message.  Members may repeat a
 * device (several streams of one GPU).  salt_group_issue_times reports, for
 * the last call, each member's issue start / end in ns after the job was
 * published (the cross-device issue skew). */
int salt_group_create(int G, const int* devices, void** group_out);
int salt_group_destroy(void* group);
int salt_group_size(void* group);
int salt_group_fused(void* group, int dtype, const char* assign_sigs, const char* reduce_sig,
                     void* const* dsts, int ndst, const void* const* leaves, int nleaves,
                     const double* scalars, int nscalars, const void* const* pscalars, int npscalars,
                     const int64_t* ns, int flags, void* const* ws, size_t ws_bytes,
                     void* const* out_dev, void* const* streams);
int salt_group_issue_times(void* group, int64_t* start_ns, int64_t* end_ns);
/* salt_group_fused with the reduction's total exchanged IN-KERNEL between the
 * members over peer memory (salt_fused_exchange per member): exchanges[i] is
 * member i's descriptor (rank i of world G; its slots / flags point at every
 * member's buffer, reachable after salt_enable_peer_access).  Every member
 * ends with the same total in out_dev[i] — one launch per device, no NCCL. */
int salt_group_fused_exchange(void* group, int dtype, const char* assign_sigs, const char* reduce_sig,
                              void* const* dsts, int ndst, const void* const* leaves, int nleaves,
                              const double* scalars, int nscalars, const void* const* pscalars,
                              int npscalars, const int64_t* ns, int flags, void* const* ws,
                              size_t ws_bytes, const salt_exchange* exchanges, void* const* out_dev,
                              void* const* streams);
/* cudaDeviceEnablePeerAccess between every pair of the G devices (already
 * enabled pairs are fine); SALT_ECUDA if a pair cannot reach each other. */
int salt_enable_peer_access(int G, const int* devices);

/* Batched assignments: `count` independent evaluations of ONE tree shape
 * `sig` (single root, no device scalars) over different vectors, scalars
 * and lengths, in ONE kernel launch per up to 96 problems (the problem table
 * travels in the kernel parameters) — for launch-bound sizes, where a launch
 * per tree costs more than its work.  leaves: count x nleaves pointers
 * (problem-major); scalars: count x nscalars; ns: count lengths.  Problems
 * must not overlap each other's destinations (they run concurrently); each
 * result has the bits of its own salt_assign.  Trees with more than 8 leaves
 * or 8 scalars run one launch per problem. */
int salt_assign_batch(int dtype, const char* sig, int count, void* const* dsts,
                      const void* const* leaves, int nleaves, const double* scalars, int nscalars,
                      const int64_t* ns, void* stream);

/* Batched small reductions: `count` independent sums of ONE reduce tree
 * `sig` over different vectors / scalars / lengths.  Problems of at most two
 * tiles (a few thousand elements) whose operands share one 32-byte
 * alignment run as ONE launch per up to 96 of them, one CTA each; the rest
 * run as ordinary reductions (workspace: salt_reduce_workspace_bytes(), used
 * only by those).  outs[q]: device pointer receiving problem q's result
 * (element type, or the {hi, lo} partial with SALT_PARTIAL; SALT_SQRT as in
 * salt_reduce).  Every result has the bits of its own salt_reduce. */
int salt_reduce_batch(int dtype, const char* sig, int count, const void* const* leaves, int nleaves,
                      const double* scalars, int nscalars, const int64_t* ns, int flags,
                      void* const* outs, void* workspace, size_t workspace_bytes, void* stream);

/* Host-buffer (end-to-end) variants: leaves / dst are HOST pointers (pinned
 * memory for full speed).  Chunks are streamed H2D -> fused kernel -> D2H
 * through `staging` (device memory, caller-owned) on three caller streams
 * so PCIe traffic in both directions overlaps the kernels.  Blocking. */
int salt_assign_host(int dtype, const char* sig, void* host_dst,
                     const void* const* host_leaves, int nleaves,
                     const double* scalars, int nscalars, int64_t n,
                     void* staging, size_t staging_bytes,
                     void* const* streams3);

int salt_reduce_host(int dtype, const char* sig,
                     const void* const* host_leaves, int nleaves,
                     const double* scalars, int nscalars, int64_t n, int flags,
                     void* staging, size_t staging_bytes,
                     void* const* streams3, void* out_host);

/* Host-buffer fused assign + reduce (salt_assign_reduce on host vectors). */
int salt_assign_reduce_host(int dtype, const char* assign_sig, const char* reduce_sig,
                            void* host_dst, const void* const* host_leaves, int nleaves,
                            const double* scalars, int nscalars, int64_t n, int flags,
                            void* staging, size_t staging_bytes,
                            void* const* streams3, void* out_host);

/* Bytes of device scratch salt_reduce / salt_assign_reduce need.  Only the
 * first SALT_WORKSPACE_TICKET_BYTES (arrival counters and collector slots)
 * must be zero before the first use; the kernels leave them zero again after
 * every reduction. */
#define SALT_WORKSPACE_TICKET_BYTES 1065216
size_t salt_reduce_workspace_bytes(void);
/* Two-step host result for callers that release a lock while waiting:
 * enqueue the device->host copy of a reduction result (out_dev, <= 64
 * bytes) into this host thread's pinned slot on `stream` and return the
 * slot; after salt_stream_synchronize(stream) the slot holds the bytes. */
int salt_result_enqueue(const void* out_dev, size_t bytes, void* stream, void** host_slot);
/* One step less: this host thread's 64-byte pinned result slot, mapped into
 * every device's address space at the same address.  Pass it as out_dev of
 * a reduction and the kernel stores the result straight into host memory:
 * after salt_stream_synchronize(stream) the slot holds it — no copy is
 * enqueued (lv.dot at n = 1024: 18.1 -> 13 us per synchronising call).
 * Fails (SALT_EINVAL) when the pool is exhausted (more than 256 host
 * threads) or the platform does not map it at the host address; callers
 * then use salt_result_enqueue.  (salt_reduce and the other reducing calls
 * do the same on their own when given out_host: the kernel stores a second
 * copy of the result into the slot, and the call only waits for the stream.) */
int salt_result_slot(void** host_slot);
int salt_stream_synchronize(void* stream);
/* Device-observed trace (debug): while a buffer is set for this host thread,
 * every salt_assign / salt_reduce / salt_fused call runs the NVRTC build of
 * its tree compiled with -DSALT_TRACE, which records the events of ONE
 * thread (thread 0 of the first streaming CTA) into trace_dev (int64):
 * word 0 = event count, then (kind, element index, slot) triples — kind 0
 * load (a slot's leaf vectors issued), 1 vector_op, 2 store, 3 single_op
 * (a scalar head/tail element), 4 reduction (the CTA's partial is formed).
 * The results are the same bits as the untraced kernel.  The buffer must be
 * zeroed before the call.  trace_dev NULL turns tracing off. */
int salt_set_trace(void* trace_dev, int64_t capacity);
/* Identity of the CUDA graph capture in progress on `stream` (0: the stream
 * is not capturing).  A reduction captured into a graph needs a workspace
 * of its own (its tickets and partials are baked into the graph): hosts key
 * per-capture workspaces by this id. */
uint64_t salt_capture_id(void* stream);

/* 0 = invalid signature, 1 = compiled-in (AOT) kernel, 2 = needs the NVRTC
 * JIT.  kind: 0 assign, 1 reduce, 2 assign+reduce (reduce_sig used). */
int salt_signature_kind(int dtype, const char* sig, const char* reduce_sig, int kind);

/* Compile (without launching) the kernels for a signature: the AOT table
 * entry if there is one, else NVRTC for both the vector and the scalar-lane
 * variant, and cache them.  Needs no GPU.  Same `kind` as above. */
int salt_prepare(int dtype, const char* sig, const char* reduce_sig, int kind);

/* Force (1) or forbid (0) the JIT for signatures that also have an AOT
 * kernel; default 0.  Used by tests to prove AOT == JIT bit for bit. */
void salt_set_force_jit(int on);
/* Test hook: evaluate every tree with the postfix interpreter kernel (the
 * fallback used when a tree is neither compiled in nor JIT-compilable, e.g.
 * without NVRTC).  salt_interp_launch_count() counts its launches. */
void salt_set_force_interp(int on);
uint64_t salt_interp_launch_count(void);
/* Tiered JIT (opt-in: SALT_JIT_ASYNC=1 or salt_set_jit_async(1); default
 * off — fresh trees are built synchronously on first use and no background
 * thread exists): a tree outside the compiled-in table and the JIT disk
 * cache runs on the interpreter kernel — same bits — while a background
 * thread compiles it with NVRTC; later calls use the compiled kernel.
 * salt_jit_wait() blocks until no compile is queued or running and returns
 * how many failed. */
void salt_set_jit_async(int on);
int salt_jit_wait(void);

/* Number of kernels this library has launched since load (all devices). */
uint64_t salt_launch_count(void);

/* Thread-local description of the last failure on this thread. */
const char* salt_last_error(void);

int salt_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* SALT_H */
