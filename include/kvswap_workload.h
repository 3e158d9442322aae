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
 * (wrapping over `buf_bytes`), on `stream`, with `ctas` CTAs (0 = 2 x SM
 * count).  `sink` (device, 16 B) receives a value only the compiler cannot
 * prove dead.  Returns 0, a KVS_ERR_* code or a cudaError_t. */
int kvs_stream_read(int device, uint64_t stream, const void* buf, size_t buf_bytes,
                    size_t bytes, int ctas, void* sink);

#ifdef __cplusplus
}
#endif

#endif /* KVSWAP_WORKLOAD_H_ */
