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
typedef struct KvsHandle KvsHandle;
int kvs_kv_tokens(KvsHandle* h, int mode, const int64_t* segs, int32_t n_segs,
                  int32_t block_tokens, int32_t plane_lo, int32_t plane_hi, uint64_t stream,
                  uint32_t* mismatch);

#ifdef __cplusplus
}
#endif

#endif /* KVSWAP_WORKLOAD_H_ */
