/*
 * ORACLE — test/bench infrastructure only (the CPU baseline, never the product).
 *
 * C restatement of one SwapPlan's byte movement, the same TransferOp
 * semantics as oracle/bytes_oracle.py::apply_plan (reference:
 * pkg/src/kvswitch/cpu_store.py:73-120 for the op list, swap.py:170-179 for
 * the op walk): for every op (blocks, gpu_start, cpu_start), block i of the op
 * maps GPU block gpu_start+i of every plane to host block cpu_start+i, whose
 * image is block-major [plane][chunk].  "GPU planes" here are ordinary host
 * buffers: this is what a CPU-only implementation of the path costs on the
 * box's own cores.  Work is split over `nthreads` pthreads by (block, plane)
 * chunk, contiguous ranges per thread.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int dir; /* 0 = out (planes -> host), 1 = in (host -> planes) */
  const uint64_t* planes;
  int num_planes;
  int64_t chunk;
  int64_t stride;
  uint8_t* host;
  const int64_t* op_end; /* inclusive prefix sums of blocks */
  const int32_t* ops;
  int32_t n_ops;
  int64_t lo, hi; /* chunk range [lo, hi) */
} Work;

static void* worker(void* arg) {
  Work* w = (Work*)arg;
  const int64_t hblk = w->chunk * w->num_planes;
  int32_t op = 0;
  for (int64_t u = w->lo; u < w->hi; ++u) {
    const int64_t k = u / w->num_planes;
    const int plane = (int)(u - k * w->num_planes);
    while (k >= w->op_end[op]) ++op;
    const int64_t begin = op ? w->op_end[op - 1] : 0;
    const int64_t rel = k - begin;
    uint8_t* g = (uint8_t*)(uintptr_t)w->planes[plane] + (w->ops[3 * op + 1] + rel) * w->stride;
    uint8_t* h = w->host + (w->ops[3 * op + 2] + rel) * hblk + plane * w->chunk;
    if (w->dir == 0)
      memcpy(h, g, (size_t)w->chunk);
    else
      memcpy(g, h, (size_t)w->chunk);
  }
  return NULL;
}

/* Returns 0 on success, -1 on bad arguments. */
int oracle_apply_plan(int dir, const uint64_t* planes, int num_planes, int64_t chunk,
                      int64_t stride, uint8_t* host, const int32_t* ops, int32_t n_ops,
                      int nthreads) {
  if ((dir != 0 && dir != 1) || num_planes < 1 || chunk < 1 || n_ops < 0 || nthreads < 1)
    return -1;
  if (n_ops == 0) return 0;
  int64_t* op_end = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_ops);
  if (!op_end) return -1;
  int64_t run = 0;
  for (int32_t i = 0; i < n_ops; ++i) {
    if (ops[3 * i] < 1) {
      free(op_end);
      return -1;
    }
    run += ops[3 * i];
    op_end[i] = run;
  }
  const int64_t units = run * num_planes;
  if (nthreads > units) nthreads = (int)units;
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
  Work* work = (Work*)malloc(sizeof(Work) * (size_t)nthreads);
  if (!tids || !work) {
    free(op_end);
    free(tids);
    free(work);
    return -1;
  }
  for (int t = 0; t < nthreads; ++t) {
    Work w = {dir, planes, num_planes, chunk, stride, host, op_end, ops, n_ops,
              units * t / nthreads, units * (t + 1) / nthreads};
    work[t] = w;
  }
  for (int t = 1; t < nthreads; ++t) pthread_create(&tids[t], NULL, worker, &work[t]);
  worker(&work[0]);
  for (int t = 1; t < nthreads; ++t) pthread_join(tids[t], NULL);
  free(op_end);
  free(tids);
  free(work);
  return 0;
}
