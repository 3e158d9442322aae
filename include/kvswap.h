/*
 * kvswap.h — C ABI of the B200 KV-swap data plane (libkvswap.so).
 *
 * The reference (kvswitch, FastSwitch arXiv 2411.18424) has no FFI: its swap
 * "data plane" is the timing model inside SwapManager.dispatch
 * (pkg/src/kvswitch/swap.py:181-232) driven by TransferOp lists
 * (pkg/src/kvswitch/cpu_store.py:73-92).  Every entry point below is what a
 * maintainer binds *underneath* that method (see INTEGRATION.md for the
 * ctypes stub); each one names the reference interface it replaces.
 *
 * Conventions
 *  - All functions return int: 0 = KVS_OK, > 0 = a cudaError_t, < 0 = a
 *    KVS_ERR_* library code.  kvs_error_string() renders either kind.
 *  - No torch / CUDA types in signatures: streams are passed as uint64_t
 *    (the value of cudaStream_t / torch.cuda.Stream.cuda_stream), device and
 *    host addresses as plain pointers / uint64_t.
 *  - Ops are the reference's TransferOp triples, flattened as int32
 *    [blocks, gpu_start, cpu_start] × n_ops (cpu_store.py:73-79).
 *  - Direction: KVS_DIR_OUT = swap-out (HBM -> pinned host, "out" in
 *    SwapPlan.direction), KVS_DIR_IN = swap-in (host -> HBM, "in").
 *
 * Geometry (one handle per GPU / TP rank):
 *  The rank's paged KV cache is `num_planes` device "planes".  A plane is one
 *  contiguous array of per-block chunks: block b of plane p lives at
 *  plane_ptrs[p] + b * plane_block_stride and is plane_chunk_bytes long.
 *  FlashInfer/vLLM-v1 per-layer [num_blocks, 2, 16, H, d] tensors are one plane
 *  per layer; split-K/V [2, num_blocks, ...] layouts are two planes per layer.
 *  The host pool is block-major: host block c is one contiguous extent of
 *  num_planes * plane_chunk_bytes bytes (plane p at offset p * chunk), so a
 *  host block group (cpu_store.py:134, a BlockGroupPool over host blocks) is
 *  one contiguous byte range and swap-out writes long sequential PCIe runs.
 */
#ifndef KVSWAP_H_
#define KVSWAP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVS_ABI_VERSION 1

#define KVS_OK 0
#define KVS_ERR_INVALID (-1)   /* bad argument (reference: ValueError)              */
#define KVS_ERR_RANGE (-2)     /* op outside a pool (reference: PoolError/IndexError) */
#define KVS_ERR_ALIGN (-3)     /* pointer/size not 16-byte aligned                   */
#define KVS_ERR_NOMEM (-4)     /* host allocation / pinning failed                   */
#define KVS_ERR_UNSUPPORTED (-5) /* driver lacks a required feature                  */

#define KVS_DIR_OUT 0
#define KVS_DIR_IN 1

/* kvs_memcpy_baseline modes (copy-engine comparators). */
#define KVS_BASE_PER_BLOCK 0 /* vLLM: one cudaMemcpyAsync per (plane, block)      */
#define KVS_BASE_PER_RUN 1   /* block groups on the CE: one cudaMemcpy2DAsync per (plane, op) */
#define KVS_BASE_STAGED 2    /* staged: one large contiguous host copy per slot of
                                a 128 MiB-slot HBM staging ring + a device gather/scatter
                                kernel between the ring and the planes            */

/* Kernel paths (kvs_set_path). */
#define KVS_PATH_LSU 0  /* v1: warps move 16-B vectors with LDG/STG (default)       */
#define KVS_PATH_BULK 1 /* v2: TMA bulk copies (cp.async.bulk) through an smem ring */

/* kvs_host_alloc flags */
#define KVS_HOST_DEFAULT 0
#define KVS_HOST_REGISTER 1 /* mmap + (optional) mbind + cudaHostRegister instead of cudaHostAlloc */
#define KVS_HOST_WRITE_COMBINED 2 /* cudaHostAlloc(...|WriteCombined): not snooped over PCIe;
                                     slow for CPU reads (the pool is GPU-only traffic) */

typedef struct KvsGeometry {
  int32_t num_planes;         /* P >= 1                                        */
  int32_t reserved;           /* must be 0                                     */
  int64_t plane_chunk_bytes;  /* bytes of one block in one plane, % 16 == 0    */
  int64_t plane_block_stride; /* bytes between blocks in a plane, >= chunk, %16 */
} KvsGeometry;

typedef struct KvsHandle KvsHandle;

/* ABI version of the loaded library (== KVS_ABI_VERSION). */
int kvs_abi_version(void);

/* Human-readable text for any return code. Never NULL. */
const char* kvs_error_string(int code);

/* Create a data-plane handle for one device (one TP rank).
 * Replaces: the bytes_per_block-only geometry SwapManager keeps
 * (swap.py:141-145, core.py:27-38); it borrows every pointer, owns none.
 * plane_ptrs: host array of num_planes device addresses (16-B aligned).
 * host_base: device-usable address of the mapped pinned host pool
 *            (num_cpu_blocks * num_planes * chunk bytes). */
int kvs_create(int device, const KvsGeometry* geo, const uint64_t* plane_ptrs,
               void* host_base, int64_t num_gpu_blocks, int64_t num_cpu_blocks,
               KvsHandle** out);

int kvs_destroy(KvsHandle* h);

/* Launch shape of the gather/scatter kernel for one direction.
 * ctas: persistent CTAs (0 = library default); threads: per CTA (multiple of 32,
 * 0 = default).  Bounded footprint keeps decode SMs free (swap.py:256-268
 * yield analogue). */
int kvs_set_launch(KvsHandle* h, int dir, int ctas, int threads);

/* Select the kernel path for one direction.  piece_bytes / stages tune the
 * bulk path's smem ring (0 = defaults: 16 KiB x 4); ignored by the LSU path.
 * Both paths serve every entry point and publish every completion word:
 * LSU warps credit per-op / per-plane counters lazily (one system fence per
 * warp and op / plane group); the bulk path's elected thread credits on its
 * store side once the TMA stores it issued for an op / group completed
 * (cp.async.bulk.wait_group 0, then a system fence). */
int kvs_set_path(KvsHandle* h, int dir, int path, int piece_bytes, int stages);

/* Pace one direction's LSU kernel to `gbps` GB/s (0 = unpaced).  Stores to
 * host memory issued faster than PCIe drains them queue up in the XBAR/L2
 * path the decode kernels' HBM traffic shares; holding the grid to the link
 * rate keeps swap-induced decode stall bounded (north star <= 10%).
 * Replaces the reference's bounded dispatch yield (swap.py:256-268). */
int kvs_set_pace(KvsHandle* h, int dir, double gbps);

/* Release a paced direction's pieces in bursts of `burst_bytes` (0 = steady)
 * at the same mean rate: the grid moves a burst at full speed, then idles
 * until the pace catches up.  Probes whether HBM writes batched in time cost
 * decode less than the same bytes spread evenly. */
int kvs_set_pace_burst(KvsHandle* h, int dir, int64_t burst_bytes);

/* One rate budget shared by both directions of this handle (0 = none): a
 * token bucket on the GPU global timer, drawn per piece by swap-out and
 * swap-in kernels alike, so a concurrent preempt + resume cannot add up to
 * more host-link traffic than decode tolerates. */
int kvs_set_budget(KvsHandle* h, double gbps);

/* Strict priority inside the shared budget: direction `dir` (or -1 = none)
 * charges the budget without waiting for it, so the other direction gets
 * only what is left.  Serving gives swap-in priority: it gates resumption
 * (engine.py:376-384), while a swap-out's freed blocks are merely busy
 * (engine.py:609, conflicts resolved per op). */
int kvs_set_budget_priority(KvsHandle* h, int dir);

/* Reserved share of the shared budget: direction `dir` always gets at least
 * `gbps` GB/s (0 = none) - a piece goes at the earlier of its shared-budget
 * slot and its slot on a private clock at `gbps` - while its pieces still
 * charge the shared budget, so a saturating other direction gets the budget
 * minus the reservation.  Between FCFS (no share) and strict priority
 * (kvs_set_budget_priority): a resume is not starved by a burst of
 * preemptions, nor does it starve them (engine.py:376-384 vs :591-611). */
int kvs_set_budget_share(KvsHandle* h, int dir, double gbps);

/* STREAM RULE — kvs_swap, kvs_swap_ops, kvs_swap_layered, kvs_swap_signaled:
 * completion words are published through per-handle, per-direction device
 * counters (a CTA ticket, op counters, plane-group counters) that each launch
 * of that direction leaves reset for the next one.  Issue every call of one
 * direction on one handle on ONE stream (one stream per direction per
 * handle).  Two streams of the same direction could interleave their tickets
 * and publish a done / op / plane flag before all of a call's CTAs landed.
 * The two directions may use two different streams.  Need more concurrency
 * in one direction: create another handle over the same pools. */

/* Queue one SwapPlan's bytes on `stream` — asynchronous, no host blocking,
 * no allocation.  Replaces the modeled copy-engine timeline of
 * SwapManager.dispatch (swap.py:193-205, costmodel.py:29-31).
 * ops: n_ops x [blocks, gpu_start, cpu_start] (TransferOp, cpu_store.py:73-79).
 * done_flag (optional, may be NULL): device-visible uint32 (device memory or
 * mapped host) that receives `seq` with system-scope release once every byte
 * of this call has landed; pair with kvs_wait_flag for cross-stream waits
 * (reference: OpRecord.exec_done / not_before, swap.py:36-42, 186).
 * Stream rule above applies. */
int kvs_swap(KvsHandle* h, int dir, const int32_t* ops, int32_t n_ops,
             uint64_t stream, uint32_t* done_flag, uint32_t seq);

/* Layer-wise pipelined swap: same bytes as kvs_swap, moved
 * plane-major in groups of planes (kvs_set_layer_group: all blocks of group 0
 * first, ...), and plane_flags[p] (device or mapped, num_planes words)
 * receives `seq` with system-scope release as soon as p's group has fully
 * landed, so decode of layer l can start (after kvs_wait_flag(stream,
 * plane_flags + l, seq)) while later layers are still in flight.  The
 * reference swaps iteration-wise.  Stream rule above. */
int kvs_swap_layered(KvsHandle* h, int dir, const int32_t* ops, int32_t n_ops,
                     uint64_t stream, uint32_t* plane_flags, uint32_t seq);

/* Plane-major order granularity of kvs_swap_layered / plane-flagged
 * kvs_swap_signaled: planes are moved in groups of `planes` (block-major
 * inside a group), 0 = auto (>= 256 KiB of a block per group, so host reads
 * stay long).  Plane l's flag fires once every plane of its group landed. */
int kvs_set_layer_group(KvsHandle* h, int planes);

/* Op-granular completion (SURVEY §7 hard part 4): same bytes as kvs_swap;
 * op_flags[i] (device or mapped, n_ops words) receives `seq` with
 * system-scope release once TransferOp i has fully landed, and done_flag
 * (optional) once the whole plan has.  A conflicting grant or swap-in then
 * waits for the blocking op only, as the reference resolves conflicts per op
 * (swap.py:236-252, engine.py:712-719), not for the whole plan.  Counters are
 * per handle and direction: issue one direction's calls on one stream. */
int kvs_swap_ops(KvsHandle* h, int dir, const int32_t* ops, int32_t n_ops,
                 uint64_t stream, uint32_t* op_flags, uint32_t* done_flag, uint32_t seq);

/* Completion words one swap call may publish (all optional, seq-valued,
 * system-scope release).  plane_flags != NULL selects plane-major order. */
typedef struct KvsSignals {
  uint32_t* op_flags;    /* n_ops words: TransferOp i landed (kvs_swap_ops)      */
  uint32_t* plane_flags; /* num_planes words: plane p landed (kvs_swap_layered)  */
  uint32_t* done_flag;   /* one word: the whole call landed (kvs_swap)           */
  uint32_t seq;
  uint32_t reserved;     /* must be 0 */
} KvsSignals;

/* One SwapPlan with any combination of the completion words above: a resumed
 * request can join decode layer by layer (plane flags) while conflicting
 * grants still wait per TransferOp (op flags).  With plane flags the order is
 * plane-major, so a TransferOp completes only with its last plane: its op
 * flag is then published when the whole call has landed.  Replaces, together:
 * engine.py:376-384 (swap-in completion, iteration-wise in the reference,
 * PAPER.md:103-105) and swap.py:236-252 (per-op conflict resolution).
 * Stream rule above applies. */
int kvs_swap_signaled(KvsHandle* h, int dir, const int32_t* ops, int32_t n_ops,
                      uint64_t stream, const KvsSignals* sig);

/* Make `stream` wait until *flag >= value (cuStreamWaitValue32 GEQ).
 * Replaces: not_before / conflict dependencies (engine.py:712-719,
 * swap.py:236-252) as a device-side wait instead of a modeled timestamp. */
int kvs_wait_flag(uint64_t stream, const uint32_t* flag, uint32_t value);

/* Number of kernels this handle has launched (gpu_launches evidence). */
int64_t kvs_launch_count(const KvsHandle* h);

/* Copy-engine paths for the same plan: vLLM per-block, per-run 2D, and
 * staged.  Reference: split_single (swap.py:170-179) is the per-block mode;
 * block groups (alloc.py) are the per-run mode.
 *
 * KVS_BASE_STAGED is a product path, not only a comparator.  SM- and
 * TMA-issued host traffic leaves in 128 B PCIe TLPs, which caps the kernels
 * near 53 GB/s.  The copy engines use larger TLPs.  But a host block image is
 * [plane][chunk] while HBM holds one plane per layer, so a direct copy is
 * chunk-sized.  The staged mode therefore splits the work:
 *   - the copy engine moves each run of adjacent host blocks as ONE
 *     contiguous copy (up to a slot, 128 MiB) between the host pool and a
 *     ring of HBM staging slots, on `stream`;
 *   - a gather (out) / scatter (in) kernel moves the slot's blocks between
 *     the ring and the planes at HBM speed, on a per-direction auxiliary
 *     stream of the handle, joined to `stream` with events.
 * Completion is stream-ordered: work queued on `stream` after the call sees
 * every byte.  The ring is allocated on first use (kvs_set_staging).  One
 * stream per direction per handle, as for kvs_swap. */
int kvs_memcpy_baseline(KvsHandle* h, int dir, int mode, const int32_t* ops,
                        int32_t n_ops, uint64_t stream);

/* Staging ring of KVS_BASE_STAGED, per direction: `slots` (2..16) slots of
 * `slot_bytes` (rounded down to whole blocks, at least one block).  0 keeps
 * the default (4 x 128 MiB).  Frees the current ring (synchronising with its
 * users) so the next staged call reallocates it. */
int kvs_set_staging(KvsHandle* h, int64_t slot_bytes, int slots);

/* Spatial SM partition for the swap kernels (green contexts): the swap side
 * gets a group of >= swap_sms SMs (rounded up to the architecture's
 * granularity, 8 on sm_90+) and the rest of the device's SMs form the
 * compute side; n_swap_streams (1..16) non-blocking streams on the swap side
 * and one on the compute side (CUstream values as uint64_t, usable with
 * kvs_swap* / any kernel launch), sms_out[0..1] = SMs per side.  Kernels in one side never run on the other's SMs, so SM-issued
 * host reads stop sharing SMs with decode CTAs.  Replaces: the reference's
 * dispatch yield bound (swap.py:256-268) as a spatial rather than temporal
 * bound.  Lives until process exit. */
int kvs_sm_partition(int device, int swap_sms, int n_swap_streams, int swap_priority,
                     int rest_priority, uint64_t* swap_streams, uint64_t* rest_stream,
                     int* sms_out);

/* Pinned, device-mapped host pool (CpuStore's backing bytes,
 * cpu_store.py:126-141).  numa_node < 0: no binding.  *dev receives the
 * device-usable address (== *host under UVA). */
int kvs_host_alloc(size_t bytes, int numa_node, int flags, void** host, void** dev);
int kvs_host_free(void* host);

#ifdef __cplusplus
}
#endif

#endif /* KVSWAP_H_ */
