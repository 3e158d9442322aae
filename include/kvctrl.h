/*
 * kvctrl.h — C ABI of the native control plane (libkvctrl.so), SURVEY §8(f)
 * rank 3: the Dynamic Block Group Manager and the CPU store with KV reuse
 * in C++, behind the reference's Python API (paper_2411_18424_b200/
 * native_ctrl.py mirrors kvswitch.alloc.BlockGroupPool and
 * kvswitch.cpu_store.CpuStore on top of it).
 *
 * Every decision — group ids, block tables, victims (including the numpy
 * PCG64 draws of the random victim policy), plans, evictions — is bit-exact
 * with the reference and with the package's Python control plane
 * (tests/test_native_ctrl.py: differential fuzz, the reference's own unit
 * tests, the engine replay goldens).
 *
 * Conventions
 *  - Host-only, single-threaded per handle, no CUDA.  All ints are int64
 *    (block indices, group ids, request ids).  "None" is KVC_NONE.
 *  - Every function returns 0 or a KVC_ERR_* code; kvc_last_error() gives the
 *    message of the last failure on the calling thread.  Codes map 1:1 onto
 *    the reference's exception classes (alloc.py:21-30, cpu_store.py:19-28).
 *  - Variable-length results are written into the handle's scratch buffer
 *    and returned as (pointer, length in int64 words); they stay valid until
 *    the next call on the same handle.
 *  - GPU extents are the block table in logical order: int64 pairs
 *    (start, length) (engine.py:317-325).  A plan is returned as
 *    [moved, reused, n_ops, n_refresh, ops (n_ops x 3), refresh (n_refresh x 3)]
 *    with each op (blocks, gpu_start, cpu_start) — the TransferOp triple the
 *    data plane (kvswap.h kvs_swap) consumes (cpu_store.py:73-92).
 */
#ifndef KVCTRL_H_
#define KVCTRL_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVC_ABI_VERSION 1
#define KVC_NONE INT64_MIN

#define KVC_OK 0
#define KVC_ERR_POOL (-10)         /* alloc.PoolError                          */
#define KVC_ERR_OOM (-11)          /* alloc.OutOfMemoryError                   */
#define KVC_ERR_NO_VICTIM (-12)    /* alloc.NoVictimError                      */
#define KVC_ERR_VALUE (-13)        /* ValueError                               */
#define KVC_ERR_KEY (-14)          /* KeyError (unknown group id)              */
#define KVC_ERR_ASSERT (-15)       /* AssertionError (validate, plan balance)  */
#define KVC_ERR_CPU_OOM (-16)      /* cpu_store.CpuOutOfMemoryError            */
#define KVC_ERR_CONTAMINATED (-17) /* cpu_store.ContaminatedCopyError          */
#define KVC_ERR_INSUFFICIENT (-18) /* cpu_store.InsufficientVictimsError       */
#define KVC_ERR_UNCOVERED (-19)    /* StopIteration: logical block not covered */

#define KVC_VICTIM_RANDOM 0
#define KVC_VICTIM_LOWEST_PRIORITY 1

typedef struct KvcPool KvcPool;
typedef struct KvcStore KvcStore;
/* Priority rank of a request (lower = more important); alloc.py:310-315. */
typedef int64_t (*kvc_rank_fn)(void* ctx, int64_t req);

int kvc_abi_version(void);
const char* kvc_last_error(void);

/* numpy-compatible PCG64 stream seeded by SeedSequence(entropy) — the
 * allocator's victim RNG (alloc.py:101).  Test hook: draws n values of
 * Generator.integers(bound) into out. */
int kvc_rng_draws(const int64_t* entropy, int32_t n_entropy, int64_t bound, int64_t n,
                  int64_t* out);

/* ---- BlockGroupPool (alloc.py:95-532) ---------------------------------- */
int kvc_pool_create(int64_t total_blocks, int64_t initial_group_blocks, int64_t rng_seed,
                    int victim_policy, KvcPool** out);
int kvc_pool_destroy(KvcPool* p);
int kvc_pool_set_rank_fn(KvcPool* p, kvc_rank_fn fn, void* ctx);
/* allocate (alloc.py:218-308): result = [n_groups, n_carved,
 * groups (id, start, length) x n_groups, carved (owner, group id) x n_carved] */
int kvc_pool_allocate(KvcPool* p, int64_t req, int64_t want, int64_t expected_total,
                      int reclaim, const int64_t** res, int64_t* len);
/* reclaim_from_victim (alloc.py:347-362): result = [owner, id, start, length] */
int kvc_pool_reclaim_from_victim(KvcPool* p, int64_t need, int64_t for_request,
                                 const int64_t** res, int64_t* len);
/* allocate_at (alloc.py:364-385): result = [] (no grant) or [id, start, length] */
int kvc_pool_allocate_at(KvcPool* p, int64_t req, int64_t start, int64_t length,
                         const int64_t** res, int64_t* len);
int kvc_pool_free_group(KvcPool* p, int64_t gid);
int kvc_pool_shrink_group(KvcPool* p, int64_t gid, int64_t new_length);
int kvc_pool_free_request(KvcPool* p, int64_t req, int64_t* freed);
int kvc_pool_set_request_fill(KvcPool* p, int64_t req, int64_t filled_blocks);
int kvc_pool_record_transfer(KvcPool* p, int64_t blocks);
/* counters: [total, free, used, groups, ops_recorded, blocks_recorded] */
int kvc_pool_counters(KvcPool* p, int64_t* out6);
int kvc_pool_owned_blocks(KvcPool* p, int64_t req, int64_t* out);
int kvc_pool_reclaimable_blocks(KvcPool* p, int64_t exclude, int64_t* out);
/* group records are 7 words: id, start, length, free, owner, active, filled */
int kvc_pool_group(KvcPool* p, int64_t gid, int64_t* out7);
int kvc_pool_owned_groups(KvcPool* p, int64_t req, const int64_t** res, int64_t* len);
int kvc_pool_free_groups(KvcPool* p, const int64_t** res, int64_t* len);
/* the block table of `req`: owned groups in grant order fused where
 * physically adjacent, (start, length) pairs (engine.py:317-325) */
int kvc_pool_extents(KvcPool* p, int64_t req, const int64_t** res, int64_t* len);
int kvc_pool_set_group_filled(KvcPool* p, int64_t gid, int64_t filled);
/* granularity histogram: (blocks, count) pairs, ascending blocks */
int kvc_pool_granularity(KvcPool* p, const int64_t** res, int64_t* len);
/* dump (alloc.py:482-490) into buf (NUL-terminated); *need = bytes required */
int kvc_pool_dump(KvcPool* p, char* buf, int64_t cap, int64_t* need);
int kvc_pool_validate(KvcPool* p);

/* ---- CpuStore (cpu_store.py:123-403) ------------------------------------ */
int kvc_store_create(int64_t total_blocks, int reuse_enabled, int64_t prealloc_min_blocks,
                     int64_t prealloc_max_blocks, int release_on_swap_in,
                     int64_t block_size_tokens, KvcStore** out);
int kvc_store_destroy(KvcStore* s);
/* the store's host block pool (borrowed; lives as long as the store) */
int kvc_store_pool(KvcStore* s, KvcPool** out);
int kvc_store_set_flag(KvcStore* s, int which, int64_t value);  /* 0 reuse, 1 refresh_dirty_tail, 2 release_on_swap_in */
/* counters: [peak_used_blocks, refreshed_blocks, n_copies, n_ranks, refresh_dirty_tail] */
int kvc_store_counters(KvcStore* s, int64_t* out5);
int kvc_store_set_rank(KvcStore* s, int64_t req, int64_t rank);
int kvc_store_set_ranks(KvcStore* s, const int64_t* pairs, int64_t n); /* (req, rank) x n */
int kvc_store_get_rank(KvcStore* s, int64_t req, int64_t* rank); /* KVC_NONE when unranked */
int kvc_store_del_rank(KvcStore* s, int64_t req);
int kvc_store_ranks(KvcStore* s, const int64_t** res, int64_t* len); /* (req, rank) pairs */
int kvc_store_clear_ranks(KvcStore* s);
/* plan_swap_out (cpu_store.py:209-287 + dirty-tail refresh); tokens KVC_NONE = unknown */
int kvc_store_plan_swap_out(KvcStore* s, int64_t req, int64_t footprint, const int64_t* extents,
                            int64_t n_extents, int64_t tokens, const int64_t** res, int64_t* len);
int kvc_store_plan_swap_in(KvcStore* s, int64_t req, const int64_t* extents, int64_t n_extents,
                           const int64_t** res, int64_t* len);
/* plan_swap_in_prefix (cpu_store.py:300-325): plan words then the kept blocks last */
int kvc_store_plan_swap_in_prefix(KvcStore* s, int64_t req, const int64_t* extents,
                                  int64_t n_extents, const int64_t** res, int64_t* len);
/* evict_for (cpu_store.py:339-385): (owner, group id) pairs taken */
int kvc_store_evict_for(KvcStore* s, int64_t rank, int64_t need, const int64_t** res, int64_t* len);
int kvc_store_preallocate_increment(KvcStore* s, int64_t req, int64_t expected_increment,
                                    int* ok);
int kvc_store_release(KvcStore* s, int64_t req);
/* _ensure_free (cpu_store.py:193-205): evict lower priorities until `need` blocks are free */
int kvc_store_ensure_free(KvcStore* s, int64_t req, int64_t need);
int kvc_store_track_peak(KvcStore* s);
/* copies: request ids holding a copy (creation order) */
int kvc_store_copy_ids(KvcStore* s, const int64_t** res, int64_t* len);
/* one copy: [prealloc, saved_tokens, n_segments, (lo, hi, group id, valid) x n]
 * (KVC_ERR_KEY when absent) */
int kvc_store_copy(KvcStore* s, int64_t req, const int64_t** res, int64_t* len);
/* replace a copy (creating it): segments (lo, hi, group id, valid) x n */
int kvc_store_put_copy(KvcStore* s, int64_t req, int64_t prealloc, int64_t saved_tokens,
                       const int64_t* segs, int64_t n_segs);
int kvc_store_drop_copy(KvcStore* s, int64_t req);

#ifdef __cplusplus
}
#endif

#endif /* KVCTRL_H_ */
