/*
 * kvswap_workload.h — synthetic decode workload exported by libkvswap.so.
 *
 * Not part of the reference's interface: the reference charges decode as
 * InferParams time (costmodel.py:34-44, iteration_time costmodel.py:74-82).
 * The live engine (paper_2411_18424_b200/live.py) replaces that number with
 * real HBM traffic of the same duration — an LLM decode step is dominated by
 * streaming the weights — so swap kernels and decode contend
 * for SMs, L2 and HBM exactly as they would in serving, and swap-induced
 * decode stall can be measured (BASELINE.json north_star: <= 10%).
 */
#ifndef KVSWAP_WORKLOAD_H_
#define KVSWAP_WORKLOAD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Stream-read `bytes` of device memory of `device` starting at `buf`
 * (wrapping over `buf_bytes`), on `stream`, with `ctas` persistent CTAs
 * (0 = 2 x SM count; each CTA owns a fixed 1/ctas share, so the step is as
 * slow as its slowest SM), or, for ctas < 0, one CTA per -ctas KiB tile
 * (thousands of CTAs that the block scheduler balances across SMs).  `sink` (device, 16 B) receives a value only the compiler cannot
 * prove dead.  Returns 0, a KVS_ERR_* code or a cudaError_t. */
int kvs_stream_read(int device, uint64_t stream, const void* buf, size_t buf_bytes,
                    size_t bytes, int ctas, void* sink);

/* Synthetic KV producer / checker: for every token of `n_segs` segments
 * (int64 x4 each: request, first token, end token, physical block holding the
 * first token; a segment's tokens sit in physically consecutive blocks of
 * `block_tokens` slots), write (mode 0) or compare (mode 1) the token's
 * deterministic K and V rows in planes [plane_lo, plane_hi) (plane_hi = -1:
 * all) of `h`'s paged cache ([2][block_tokens][row] per plane chunk), on
 * `stream`.  Mode 0 stands in for the KV attention appends each iteration;
 * mode 1 for attention reading the batch's KV, adding the number of
 * differing 32-bit words to *mismatch (device memory).  Word w of plane p, K/V kv of
 * token t of request r is t*0x01000193 + r*0x5BD1E995 + p*0x9E3779B1 +
 * kv*0x7F4A7C15 + w (mod 2^32). */
/* kvs_stream_read with launch flags: KVS_DECODE_PDL launches with
 * programmatic stream serialization and triggers the next kernel's launch at
 * entry (a CUDA-graph / PDL decode, as serving engines chain a model's
 * per-layer kernels); KVS_DECODE_WAIT then waits (griddepcontrol.wait) for
 * the previous kernel's completion before reading — a real layer-to-layer
 * dependency, so only launch latency and ramp overlap, not the work. */
#define KVS_DECODE_PDL 1
#define KVS_DECODE_WAIT 2
int kvs_stream_read_ex(int device, uint64_t stream, const void* buf, size_t buf_bytes,
                       size_t bytes, int ctas, void* sink, int flags);

/* Decode step as a CUDA graph (how serving engines launch a model's
 * per-layer decode kernels).  Stream-launched kernels fetch their commands
 * from host memory over the same PCIe link a swap-in saturates, so every
 * launch waits behind the swap's reads (a 32-layer step pays
 * +20% under a full-rate swap-in stream-launched, +9% graph-launched).
 *
 * kvs_graph_begin starts capturing on the graph's private stream
 * (kvs_graph_stream); launch decode kernels (kvs_stream_read(_ex),
 * kvs_kv_tokens), plane-flag waits (kvs_wait_flag) and timing marks
 * (kvs_graph_mark: event `slot` recorded as a graph node) on it;
 * kvs_graph_end ends the capture and updates the executable graph in place
 * (cudaGraphExecUpdate, *how = 1) or instantiates it (*how = 2) when the
 * step's structure changed; kvs_graph_launch runs it on `stream`.
 * kvs_graph_elapsed reads the time between two marks after the launch
 * completed.  A captured kvs_wait_flag parks its hardware queue until the
 * flag is published: queue the flag's producer (the swap) before launching
 * the step that waits for it, as the live engine does. */
typedef struct KvsGraph KvsGraph;
int kvs_graph_create(int device, int n_marks, KvsGraph** out);
int kvs_graph_destroy(KvsGraph* g);
int kvs_graph_stream(KvsGraph* g, uint64_t* stream);
int kvs_graph_begin(KvsGraph* g);
int kvs_graph_mark(KvsGraph* g, int slot);
int kvs_graph_end(KvsGraph* g, int* how);
int kvs_graph_launch(KvsGraph* g, uint64_t stream);
int kvs_graph_elapsed(KvsGraph* g, int slot_a, int slot_b, float* ms);
/* instantiations, in-place updates, launches */
int kvs_graph_stats(KvsGraph* g, int64_t* out3);

typedef struct KvsHandle KvsHandle;
int kvs_kv_tokens(KvsHandle* h, int mode, const int64_t* segs, int32_t n_segs,
                  int32_t block_tokens, int32_t plane_lo, int32_t plane_hi, uint64_t stream,
                  uint32_t* mismatch);

/* One decode step captured into `g` in one call (what the live engine did
 * with ~100 calls from Python per step: the host time a synchronous loop
 * adds to every token).  Per layer l = 0..h's planes-1:
 *   - wait until dep_flags[d][l] >= dep_seqs[d] for every dep d (plane
 *     flags of layer-pipelined swap-ins, kvs_swap_signaled);
 *   - mark 2l (if marks);
 *   - check the resident KV of `segs` in plane l (kvs_kv_tokens mode 1);
 *   - stream w_bytes_per_layer bytes of `weights` (kvs_stream_read);
 *   - mark 2l+1 (if marks).
 * Then ends the capture (kvs_graph_end semantics, *how). */
typedef struct KvsDecodeStep {
  const int64_t* segs;         /* [n_segs][4] (request, lo, hi, physical block of lo) */
  int32_t n_segs;
  int32_t block_tokens;
  uint32_t* mismatch;          /* KV check counter (required when n_segs > 0) */
  const void* weights;
  uint64_t weight_bytes;
  uint64_t w_bytes_per_layer;  /* 0: no weight streaming */
  void* sink;
  int32_t w_ctas;              /* kvs_stream_read ctas */
  int32_t n_deps;
  const uint64_t* dep_flags;   /* [n_deps] device addresses of per-plane flag arrays */
  const uint32_t* dep_seqs;    /* [n_deps] */
  int32_t marks;               /* 1: timing marks around each layer (needs 2 x planes marks) */
  int32_t reserved;            /* must be 0 */
} KvsDecodeStep;
int kvs_graph_decode_step(KvsGraph* g, KvsHandle* h, const KvsDecodeStep* step, int* how);

#ifdef __cplusplus
}
#endif

#endif /* KVSWAP_WORKLOAD_H_ */
