// libkvctrl — native control plane behind the C ABI in
// include/kvctrl.h: the Dynamic Block Group Manager (reference
// pkg/src/kvswitch/alloc.py) and the CPU store with multi-turn KV reuse
// (pkg/src/kvswitch/cpu_store.py), plus the B200 dirty-tail refresh op
// (SURVEY §0 finding 3).  Decisions are bit-exact with the reference,
// including the allocator's numpy PCG64 victim draws.
//
// Data structures (host DRAM, one handle per pool / store):
//  * groups live in a hash map by id; two ordered sets index the free groups
//    by (length, start) for best-fit / largest and by start for exact-extent
//    grants — O(log F) per decision instead of the reference's O(F) scans of
//    an unordered id set (alloc.py:258-282);
//  * start_of / end_of hash maps give O(1) neighbour lookups for coalescing;
//  * a store keeps each request's copy as a segment vector (cpu_store.py:31-70).

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <tuple>
#include <unordered_map>
#include <utility>
#include <vector>

#include "kvctrl.h"

namespace kvc {

thread_local std::string g_err;

struct Err {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, std::string msg) { throw Err{code, std::move(msg)}; }

std::string i2s(int64_t v) { return std::to_string(v); }

// ---------------------------------------------------------------------------
// numpy Generator(PCG64(SeedSequence(entropy))).integers(bound)
// ---------------------------------------------------------------------------
using u128 = unsigned __int128;

class SeedSequence {
 public:
  explicit SeedSequence(const std::vector<uint32_t>& entropy) {
    uint32_t hash_const = kInitA;
    auto hashmix = [&hash_const](uint32_t value) {
      value ^= hash_const;
      hash_const *= kMultA;
      value *= hash_const;
      value ^= value >> kXShift;
      return value;
    };
    auto mix = [](uint32_t x, uint32_t y) {
      uint32_t r = kMixMultL * x - kMixMultR * y;
      r ^= r >> kXShift;
      return r;
    };
    for (int i = 0; i < kPool; ++i)
      pool_[i] = hashmix(i < static_cast<int>(entropy.size()) ? entropy[i] : 0u);
    for (int s = 0; s < kPool; ++s)
      for (int d = 0; d < kPool; ++d)
        if (s != d) pool_[d] = mix(pool_[d], hashmix(pool_[s]));
    for (size_t s = kPool; s < entropy.size(); ++s)
      for (int d = 0; d < kPool; ++d) pool_[d] = mix(pool_[d], hashmix(entropy[s]));
  }

  // generate_state(n, uint64): 2n uint32 words, little-endian pairs
  std::vector<uint64_t> state64(int n) const {
    std::vector<uint64_t> out(n);
    uint32_t hash_const = kInitB;
    for (int i = 0; i < 2 * n; ++i) {
      uint32_t v = pool_[i % kPool];
      v ^= hash_const;
      hash_const *= kMultB;
      v *= hash_const;
      v ^= v >> kXShift;
      if (i % 2 == 0)
        out[i / 2] = v;
      else
        out[i / 2] |= static_cast<uint64_t>(v) << 32;
    }
    return out;
  }

 private:
  static constexpr int kPool = 4;
  static constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u;
  static constexpr uint32_t kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
  static constexpr uint32_t kMixMultL = 0xca01f9ddu, kMixMultR = 0x4973f715u;
  static constexpr int kXShift = 16;
  uint32_t pool_[kPool];
};

// numpy's _coerce_to_uint32_array for non-negative Python ints
std::vector<uint32_t> coerce_entropy(const int64_t* e, int n) {
  std::vector<uint32_t> out;
  for (int i = 0; i < n; ++i) {
    if (e[i] < 0) fail(KVC_ERR_VALUE, "expected non-negative integer");
    uint64_t v = static_cast<uint64_t>(e[i]);
    if (v == 0) {
      out.push_back(0);
      continue;
    }
    while (v) {
      out.push_back(static_cast<uint32_t>(v & 0xFFFFFFFFu));
      v >>= 32;
    }
  }
  return out;
}

class Pcg64 {
 public:
  void seed(const std::vector<uint32_t>& entropy) {
    const std::vector<uint64_t> s = SeedSequence(entropy).state64(4);
    const u128 initstate = (static_cast<u128>(s[0]) << 64) | s[1];
    const u128 initseq = (static_cast<u128>(s[2]) << 64) | s[3];
    state_ = 0;
    inc_ = (initseq << 1) | 1u;
    step();
    state_ += initstate;
    step();
    has32_ = false;
  }

  uint64_t next64() {
    step();
    const uint64_t hi = static_cast<uint64_t>(state_ >> 64), lo = static_cast<uint64_t>(state_);
    const unsigned rot = static_cast<unsigned>(state_ >> 122);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }

  uint32_t next32() {
    if (has32_) {
      has32_ = false;
      return buf32_;
    }
    const uint64_t v = next64();
    has32_ = true;
    buf32_ = static_cast<uint32_t>(v >> 32);
    return static_cast<uint32_t>(v);
  }

  // Generator.integers(bound): Lemire's bounded draw (numpy distributions.c)
  int64_t integers(int64_t bound) {
    if (bound < 1) fail(KVC_ERR_VALUE, "high <= 0");
    const uint64_t rng = static_cast<uint64_t>(bound) - 1;
    if (rng == 0) return 0;
    if (rng <= 0xFFFFFFFFull) {
      if (rng == 0xFFFFFFFFull) return next32();
      const uint32_t excl = static_cast<uint32_t>(rng) + 1;
      uint64_t m = static_cast<uint64_t>(next32()) * excl;
      uint32_t left = static_cast<uint32_t>(m);
      if (left < excl) {
        const uint32_t threshold = (UINT32_MAX - static_cast<uint32_t>(rng)) % excl;
        while (left < threshold) {
          m = static_cast<uint64_t>(next32()) * excl;
          left = static_cast<uint32_t>(m);
        }
      }
      return static_cast<int64_t>(m >> 32);
    }
    const uint64_t excl = rng + 1;
    u128 m = static_cast<u128>(next64()) * excl;
    uint64_t left = static_cast<uint64_t>(m);
    if (left < excl) {
      const uint64_t threshold = (UINT64_MAX - rng) % excl;
      while (left < threshold) {
        m = static_cast<u128>(next64()) * excl;
        left = static_cast<uint64_t>(m);
      }
    }
    return static_cast<int64_t>(m >> 64);
  }

 private:
  void step() {
    static const u128 kMult =
        (static_cast<u128>(2549297995355413924ull) << 64) | 4865540595714422341ull;
    state_ = state_ * kMult + inc_;
  }
  u128 state_ = 0, inc_ = 0;
  bool has32_ = false;
  uint32_t buf32_ = 0;
};

constexpr int64_t kAllocRngLabel = 0x6A11;  // alloc.py:101 stream label
constexpr int64_t kVictimHeadroom = 8;      // alloc.py:86-88

// ---------------------------------------------------------------------------
// BlockGroupPool
// ---------------------------------------------------------------------------
struct Group {
  int64_t id, start, length;
  bool free;
  int64_t owner;  // KVC_NONE when free
  bool active;
  int64_t filled;
  int64_t end() const { return start + length; }
  int64_t unused_tail() const { return length - filled; }
};

}  // namespace kvc

using namespace kvc;

struct KvcPool {
  int64_t total = 0, initial = 60;
  int victim_policy = KVC_VICTIM_RANDOM;
  Pcg64 rng;
  kvc_rank_fn rank_fn = nullptr;
  void* rank_ctx = nullptr;
  int64_t id_counter = 0;
  std::unordered_map<int64_t, Group> groups;
  std::unordered_map<int64_t, int64_t> start_of, end_of;
  std::set<std::tuple<int64_t, int64_t, int64_t>> by_size;  // (length, start, id)
  std::set<std::pair<int64_t, int64_t>> by_addr;             // (start, id)
  std::unordered_map<int64_t, std::vector<int64_t>> owned;   // grant order
  std::unordered_map<int64_t, int64_t> active;
  int64_t free_total = 0;
  std::map<int64_t, int64_t> sizes;
  int64_t ops_recorded = 0, blocks_recorded = 0;
  std::vector<int64_t> out;
  std::string text;

  // -------------------------------------------------------------- plumbing
  Group fresh(int64_t start, int64_t length, bool is_free) {
    Group g{id_counter++, start, length, is_free, KVC_NONE, false, 0};
    return g;
  }
  void free_add(const Group& g) {
    by_size.emplace(g.length, g.start, g.id);
    by_addr.emplace(g.start, g.id);
  }
  void free_drop(int64_t length, int64_t start, int64_t id) {
    by_size.erase(std::make_tuple(length, start, id));
    by_addr.erase(std::make_pair(start, id));
  }
  Group& at(int64_t gid) {
    auto it = groups.find(gid);
    if (it == groups.end()) fail(KVC_ERR_KEY, i2s(gid));
    return it->second;
  }
  void link(const Group& g) {
    groups[g.id] = g;
    start_of[g.start] = g.id;
    end_of[g.end()] = g.id;
    if (g.free) free_add(g);
  }
  Group unlink(int64_t gid) {
    Group g = at(gid);
    if (g.free) free_drop(g.length, g.start, g.id);
    groups.erase(gid);
    start_of.erase(g.start);
    end_of.erase(g.end());
    return g;
  }
  void resize(int64_t gid, int64_t start, int64_t length) {
    Group& g = at(gid);
    if (g.free) free_drop(g.length, g.start, g.id);
    auto s = start_of.find(g.start);
    if (s != start_of.end() && s->second == gid) start_of.erase(s);
    auto e = end_of.find(g.end());
    if (e != end_of.end() && e->second == gid) end_of.erase(e);
    g.start = start;
    g.length = length;
    start_of[g.start] = gid;
    end_of[g.end()] = gid;
    if (g.free) free_add(g);
  }
  Group take_front(int64_t gid, int64_t n) {
    free_total -= n;
    Group& g = at(gid);
    if (n == g.length) {
      Group whole = unlink(gid);
      whole.free = false;
      return whole;
    }
    Group piece = fresh(g.start, n, false);
    resize(gid, g.start + n, g.length - n);
    return piece;
  }
  void give(Group g, int64_t owner) {
    g.free = false;
    g.owner = owner;
    g.active = false;
    g.filled = 0;
    link(g);
    owned[owner].push_back(g.id);
  }
  void activate(int64_t owner, int64_t gid) {
    auto it = active.find(owner);
    if (it != active.end()) {
      auto prev = groups.find(it->second);
      if (prev != groups.end()) prev->second.active = false;
    }
    at(gid).active = true;
    active[owner] = gid;
  }
  static void remove_first(std::vector<int64_t>& v, int64_t x) {
    auto it = std::find(v.begin(), v.end(), x);
    if (it == v.end()) fail(KVC_ERR_VALUE, "list.remove(x): x not in list");
    v.erase(it);
  }
  void after_loss(int64_t owner, bool lost_active) {
    auto it = owned.find(owner);
    if (it == owned.end() || it->second.empty()) {
      if (it != owned.end()) owned.erase(it);
      active.erase(owner);
    } else if (lost_active) {
      activate(owner, it->second.back());
    }
  }

  // ---------------------------------------------------------------- queries
  int64_t owned_blocks(int64_t req) const {
    int64_t t = 0;
    auto it = owned.find(req);
    if (it != owned.end())
      for (int64_t gid : it->second) t += groups.at(gid).length;
    return t;
  }
  static int64_t carvable(const Group& g) {
    const int64_t tail = g.unused_tail();
    return tail > 0 ? tail - std::min(kVictimHeadroom, tail) : 0;
  }
  std::vector<Group*> victims(int64_t exclude) {
    std::vector<Group*> found;
    for (auto& kv : active) {
      if (exclude != KVC_NONE && kv.first == exclude) continue;
      Group& g = at(kv.second);
      if (g.unused_tail() > 0) found.push_back(&g);
    }
    std::sort(found.begin(), found.end(), [](const Group* a, const Group* b) {
      return a->owner != b->owner ? a->owner < b->owner : a->id < b->id;
    });
    return found;
  }
  int64_t reclaimable(int64_t exclude) {  // sum over victims(): no order needed
    int64_t t = 0;
    for (auto& kv : active) {
      if (exclude != KVC_NONE && kv.first == exclude) continue;
      const int64_t tail = at(kv.second).unused_tail();
      if (tail > 0) t += tail;
    }
    return t;
  }
  int64_t rank_of(int64_t owner) {
    return rank_fn(rank_ctx, owner);
  }
  Group* pick_victim(std::vector<Group*> cands) {
    std::sort(cands.begin(), cands.end(), [](const Group* a, const Group* b) {
      return a->owner != b->owner ? a->owner < b->owner : a->id < b->id;
    });
    if (victim_policy == KVC_VICTIM_LOWEST_PRIORITY && rank_fn != nullptr) {
      Group* best = nullptr;
      int64_t best_rank = 0;
      for (Group* g : cands) {  // max by (rank, owner); first maximum wins
        const int64_t r = rank_of(g->owner);
        if (best == nullptr || r > best_rank || (r == best_rank && g->owner > best->owner)) {
          best = g;
          best_rank = r;
        }
      }
      return best;
    }
    return cands[static_cast<size_t>(rng.integers(static_cast<int64_t>(cands.size())))];
  }

  // ------------------------------------------------------------- allocation
  void allocate(int64_t req, int64_t want, int64_t expected, bool reclaim,
                std::vector<Group>& grants, std::vector<std::pair<int64_t, int64_t>>& carved) {
    if (want < 1) fail(KVC_ERR_VALUE, "want_blocks must be >= 1, got " + i2s(want));
    // Carvable tails only matter when the free blocks fall short (the
    // reference sums them on every call, alloc.py:224-229; same decision).
    int64_t supply = free_total;
    if (reclaim && supply < want) supply += reclaimable(req);
    if (supply < want)
      fail(KVC_ERR_OOM, "need " + i2s(want) + " blocks, supply " + i2s(supply) + " (free " +
                            i2s(free_total) + ")");
    int64_t goal = want;
    if (expected != KVC_NONE && want < initial)
      goal = std::min(initial, std::max(want, expected));
    goal = std::max(want, std::min(goal, free_total));
    int64_t left = goal;
    while (left > 0) {
      auto bf = by_size.lower_bound(std::make_tuple(left, INT64_MIN, INT64_MIN));
      if (bf != by_size.end()) {
        Group piece = take_front(std::get<2>(*bf), left);
        give(piece, req);
        grants.push_back(groups.at(piece.id));
        break;
      }
      if (!by_size.empty()) {
        const int64_t top = std::get<0>(*by_size.rbegin());
        auto lg = by_size.lower_bound(std::make_tuple(top, INT64_MIN, INT64_MIN));
        const int64_t n = std::get<0>(*lg);
        Group piece = take_front(std::get<2>(*lg), n);
        give(piece, req);
        grants.push_back(groups.at(piece.id));
        left -= n;
        continue;
      }
      if (!reclaim) fail(KVC_ERR_OOM, "free supply changed mid-allocation");
      int64_t n = 0;
      Group* v = choose_carve(req, left, &n);
      carved.emplace_back(v->owner, v->id);
      grants.push_back(carve_tail(v->id, n, req));
      left -= n;
    }
    activate(req, grants.back().id);
    for (Group& g : grants) g = groups.at(g.id);  // reflect the active flag
  }
  Group* choose_carve(int64_t req, int64_t need, int64_t* n) {
    std::vector<Group*> pool = victims(req);
    std::vector<Group*> whole;
    for (Group* g : pool)
      if (g->unused_tail() >= need) whole.push_back(g);
    if (!whole.empty()) {
      *n = need;
      return pick_victim(whole);
    }
    Group* v = nullptr;
    for (Group* g : pool) {  // max by (carvable, -id)
      const int64_t c = carvable(*g);
      if (c <= 0) continue;
      if (v == nullptr || c > carvable(*v) || (c == carvable(*v) && g->id < v->id)) v = g;
    }
    if (v != nullptr) {
      *n = std::min(carvable(*v), need);
      return v;
    }
    if (pool.empty()) fail(KVC_ERR_OOM, "victim supply changed mid-allocation");
    for (Group* g : pool)  // headroom is best effort: strip whole tails
      if (v == nullptr || g->unused_tail() > v->unused_tail() ||
          (g->unused_tail() == v->unused_tail() && g->id < v->id))
        v = g;
    *n = std::min(v->unused_tail(), need);
    return v;
  }
  Group carve_tail(int64_t vid, int64_t n, int64_t new_owner) {
    Group& v = at(vid);
    if (v.free || n < 1 || n > v.unused_tail()) fail(KVC_ERR_ASSERT, "bad carve");
    if (n < v.length) {
      resize(vid, v.start, v.length - n);
      Group piece = fresh(at(vid).end(), n, false);
      give(piece, new_owner);
      return groups.at(piece.id);
    }
    const int64_t old_owner = v.owner;
    remove_first(owned[old_owner], vid);
    const bool lost_active = v.active;
    Group g = unlink(vid);
    g.id = id_counter++;
    g.active = false;
    g.owner = new_owner;
    link(g);
    owned[new_owner].push_back(g.id);
    after_loss(old_owner, lost_active);
    return groups.at(g.id);
  }
  std::pair<int64_t, Group> reclaim_from_victim(int64_t need, int64_t for_request) {
    if (need < 1) fail(KVC_ERR_VALUE, "need_blocks must be >= 1, got " + i2s(need));
    std::vector<Group*> fits;
    for (Group* g : victims(for_request))
      if (g->unused_tail() >= need) fits.push_back(g);
    if (fits.empty())
      fail(KVC_ERR_NO_VICTIM, "no active group has " + i2s(need) + " unused tail blocks");
    Group* v = pick_victim(fits);
    const int64_t owner = v->owner;
    Group piece = carve_tail(v->id, need, for_request);
    activate(for_request, piece.id);
    return {owner, groups.at(piece.id)};
  }
  bool allocate_at(int64_t req, int64_t start, int64_t length, Group* out_g) {
    if (length == 0) return false;
    auto it = by_addr.upper_bound(std::make_pair(start, INT64_MAX));
    if (it == by_addr.begin()) return false;
    --it;
    const int64_t gid = it->second;
    Group& g = at(gid);
    if (g.end() < start + length) return false;
    if (g.start < start) {
      Group lead = fresh(g.start, start - g.start, true);
      resize(gid, start, g.end() - start);
      link(lead);
    }
    Group piece = take_front(gid, length);
    give(piece, req);
    activate(req, piece.id);
    *out_g = groups.at(piece.id);
    return true;
  }

  // ---------------------------------------------------------------- release
  void free_group(int64_t gid) {
    auto it = groups.find(gid);
    if (it == groups.end() || it->second.free)
      fail(KVC_ERR_POOL, "group " + i2s(gid) + " is not allocated (double free?)");
    Group& g = it->second;
    const int64_t owner = g.owner;
    remove_first(owned[owner], gid);
    const bool lost_active = g.active;
    g.owner = KVC_NONE;
    g.active = false;
    g.filled = 0;
    free_total += g.length;
    auto li = end_of.find(g.start);
    const int64_t left_id = li != end_of.end() ? li->second : KVC_NONE;
    auto ri = start_of.find(g.end());
    const int64_t right_id = ri != start_of.end() ? ri->second : KVC_NONE;
    int64_t survivor = gid;
    if (left_id != KVC_NONE && at(left_id).free) {
      const Group gone = unlink(gid);
      Group& l = at(left_id);
      resize(left_id, l.start, l.length + gone.length);
      survivor = left_id;
    } else {
      g.free = true;
      free_add(g);
    }
    if (right_id != KVC_NONE && at(right_id).free) {
      const Group r = unlink(right_id);
      Group& s = at(survivor);
      resize(survivor, s.start, s.length + r.length);
    }
    after_loss(owner, lost_active);
  }
  void shrink_group(int64_t gid, int64_t new_length) {
    Group& g = at(gid);
    if (g.free) fail(KVC_ERR_POOL, "group " + i2s(gid) + " is free");
    if (new_length < 1 || new_length > g.length)
      fail(KVC_ERR_VALUE,
           "bad shrink target " + i2s(new_length) + " for length " + i2s(g.length));
    if (new_length == g.length) return;
    const int64_t cut = g.length - new_length;
    resize(gid, g.start, new_length);
    Group& h = at(gid);
    h.filled = std::min(h.filled, new_length);
    Group tail = fresh(h.end(), cut, true);
    free_total += cut;
    auto ri = start_of.find(tail.end());
    if (ri != start_of.end() && at(ri->second).free) {
      const Group r = unlink(ri->second);
      tail.length += r.length;
    }
    link(tail);
  }
  int64_t free_request(int64_t req) {
    int64_t freed = 0;
    auto it = owned.find(req);
    if (it == owned.end()) return 0;
    const std::vector<int64_t> ids = it->second;
    for (int64_t gid : ids) {
      freed += at(gid).length;
      free_group(gid);
    }
    return freed;
  }
  void set_request_fill(int64_t req, int64_t filled_blocks) {
    int64_t rest = filled_blocks;
    auto it = owned.find(req);
    if (it != owned.end())
      for (int64_t gid : it->second) {
        Group& g = at(gid);
        g.filled = rest < g.length ? rest : g.length;
        rest -= g.filled;
      }
    if (rest > 0)
      fail(KVC_ERR_POOL, "request " + i2s(req) + " holds fewer blocks than fill level " +
                             i2s(filled_blocks));
  }

  // -------------------------------------------------------------- debugging
  std::vector<const Group*> address_order() const {
    std::vector<std::pair<int64_t, int64_t>> starts(start_of.begin(), start_of.end());
    std::sort(starts.begin(), starts.end());
    std::vector<const Group*> out_g;
    out_g.reserve(starts.size());
    for (auto& s : starts) out_g.push_back(&groups.at(s.second));
    return out_g;
  }
  std::string dump() const {
    std::string s;
    char line[128];
    bool first = true;
    for (const Group* g : address_order()) {
      if (!first) s.push_back('\n');
      first = false;
      if (g->owner == KVC_NONE)
        snprintf(line, sizeof line, "%lld %lld %s - %d", static_cast<long long>(g->start),
                 static_cast<long long>(g->length), g->free ? "free" : "used", g->active ? 1 : 0);
      else
        snprintf(line, sizeof line, "%lld %lld %s %lld %d", static_cast<long long>(g->start),
                 static_cast<long long>(g->length), g->free ? "free" : "used",
                 static_cast<long long>(g->owner), g->active ? 1 : 0);
      s += line;
    }
    return s;
  }
  void validate() const {
    int64_t cursor = 0, free_sum = 0, n_free = 0;
    bool prev_free = false;
    for (const Group* g : address_order()) {
      if (g->start != cursor)
        fail(KVC_ERR_ASSERT,
             "gap or overlap at block " + i2s(cursor) + " (group " + i2s(g->id) + ")");
      if (g->length < 1)
        fail(KVC_ERR_ASSERT, "group " + i2s(g->id) + " has length " + i2s(g->length));
      if (g->free && prev_free) fail(KVC_ERR_ASSERT, "adjacent free groups at " + i2s(g->start));
      if (g->free != (g->owner == KVC_NONE))
        fail(KVC_ERR_ASSERT, "group " + i2s(g->id) + " free/owner mismatch");
      if (g->filled > g->length) fail(KVC_ERR_ASSERT, "group " + i2s(g->id) + " overfilled");
      if (g->free) free_sum += g->length;
      cursor = g->end();
      prev_free = g->free;
    }
    if (cursor != total)
      fail(KVC_ERR_ASSERT, "pool covers " + i2s(cursor) + " of " + i2s(total) + " blocks");
    if (groups.size() != start_of.size()) fail(KVC_ERR_ASSERT, "index size mismatch");
    for (auto& kv : groups) n_free += kv.second.free ? 1 : 0;
    if (free_sum != free_total || static_cast<int64_t>(by_addr.size()) != n_free)
      fail(KVC_ERR_ASSERT, "free-block counter out of sync");
    for (auto& kv : owned) {
      int64_t n_act = 0, act = KVC_NONE;
      for (int64_t gid : kv.second)
        if (groups.at(gid).active) {
          ++n_act;
          act = gid;
        }
      auto a = active.find(kv.first);
      if (n_act != 1 || a == active.end() || a->second != act)
        fail(KVC_ERR_ASSERT, "request " + i2s(kv.first) + " active-group invariant broken");
    }
  }

  void put(const Group& g) {
    out.insert(out.end(), {g.id, g.start, g.length, g.free ? 1 : 0, g.owner, g.active ? 1 : 0,
                           g.filled});
  }
};

// ---------------------------------------------------------------------------
// CpuStore
// ---------------------------------------------------------------------------
namespace kvc {

struct Seg {
  int64_t lo, hi, gid;  // gid KVC_NONE once another request took the space
  bool valid;
  int64_t length() const { return hi - lo; }
};

struct Copy {
  int64_t order = 0;  // creation order (dict insertion order)
  std::vector<Seg> segs;
  int64_t prealloc = KVC_NONE;
  int64_t saved = KVC_NONE;
  int64_t covered() const { return segs.empty() ? 0 : segs.back().hi; }
  bool fully_valid() const {
    for (const Seg& s : segs)
      if (!s.valid) return false;
    return true;
  }
  int64_t valid_prefix() const {
    int64_t reach = 0;
    for (const Seg& s : segs) {
      if (!(s.valid && s.lo == reach)) return reach;
      reach = s.hi;
    }
    return reach;
  }
};

struct Extent {
  int64_t lo, hi, phys;
};

struct Op {
  int64_t blocks, gpu, cpu;
};

const Extent& locate(const std::vector<Extent>& ext, int64_t pos) {
  for (const Extent& e : ext)
    if (e.lo <= pos && pos < e.hi) return e;
  fail(KVC_ERR_UNCOVERED, "logical block " + i2s(pos) + " not covered");
}

// cpu_store.py:95-120: one op per stretch contiguous on both sides
void pair_extents(const std::vector<std::pair<int64_t, int64_t>>& ranges,
                  const std::vector<Extent>& gpu, const std::vector<Extent>& cpu,
                  std::vector<Op>& ops) {
  for (auto& r : ranges) {
    int64_t pos = r.first;
    while (pos < r.second) {
      const Extent& g = locate(gpu, pos);
      const Extent& c = locate(cpu, pos);
      const int64_t stop = std::min({r.second, g.hi, c.hi});
      ops.push_back({stop - pos, g.phys + pos - g.lo, c.phys + pos - c.lo});
      pos = stop;
    }
  }
}

std::vector<Extent> gpu_logical(const int64_t* ext, int64_t n) {
  std::vector<Extent> out;
  out.reserve(static_cast<size_t>(n));
  int64_t pos = 0;
  for (int64_t i = 0; i < n; ++i) {
    out.push_back({pos, pos + ext[2 * i + 1], ext[2 * i]});
    pos += ext[2 * i + 1];
  }
  return out;
}

}  // namespace kvc

struct KvcStore {
  KvcPool pool;
  bool reuse = true, release_on_swap_in = false, refresh_dirty_tail = true;
  int64_t pmin = 8, pmax = 256, block_tokens = 16;
  std::unordered_map<int64_t, Copy> copies;
  int64_t copy_order = 0;
  std::unordered_map<int64_t, int64_t> ranks;
  int64_t peak = 0, refreshed = 0;
  std::vector<int64_t> out;

  int64_t rank_or0(int64_t req) const {
    auto it = ranks.find(req);
    return it == ranks.end() ? 0 : it->second;
  }
  void track_peak() { peak = std::max(peak, pool.total - pool.free_total); }
  int64_t drop_prealloc(Copy& c) {
    if (c.prealloc == KVC_NONE) return 0;
    const int64_t n = pool.at(c.prealloc).length;
    pool.free_group(c.prealloc);
    c.prealloc = KVC_NONE;
    return n;
  }
  std::vector<Extent> host_extents(const Copy& c) {
    std::vector<Extent> out_e;
    for (const Seg& s : c.segs) {
      if (s.gid == KVC_NONE) continue;
      const int64_t phys = pool.at(s.gid).start;
      if (!out_e.empty()) {
        Extent& e = out_e.back();
        if (e.hi == s.lo && e.phys + (e.hi - e.lo) == phys) {
          e.hi = s.hi;
          continue;
        }
      }
      out_e.push_back({s.lo, s.hi, phys});
    }
    return out_e;
  }
  void ensure_free(int64_t req, int64_t need) {
    const int64_t short_by = need - pool.free_total;
    if (short_by <= 0) return;
    try {
      evict_for(rank_or0(req), short_by, nullptr);
    } catch (const Err& e) {
      if (e.code != KVC_ERR_INSUFFICIENT) throw;
      fail(KVC_ERR_CPU_OOM, "cannot host " + i2s(need) + " blocks for request " + i2s(req));
    }
    if (pool.free_total < need)
      fail(KVC_ERR_CPU_OOM, "cannot host " + i2s(need) + " blocks for request " + i2s(req));
  }
  Copy& copy_setdefault(int64_t req) {
    auto it = copies.find(req);
    if (it != copies.end()) return it->second;
    Copy& c = copies[req];
    c.order = copy_order++;
    return c;
  }

  int64_t stale_tail(const Copy& c, int64_t footprint, int64_t tokens) const {
    if (!refresh_dirty_tail || tokens == KVC_NONE || c.saved == KVC_NONE || c.segs.empty())
      return KVC_NONE;
    const int64_t saved = c.saved;
    if (tokens <= saved || saved % block_tokens == 0) return KVC_NONE;
    const int64_t tail = saved / block_tokens;
    if (tail >= c.covered() || tail >= footprint) return KVC_NONE;
    for (const Seg& s : c.segs)
      if (s.lo <= tail && tail < s.hi) return s.valid ? tail : KVC_NONE;
    return KVC_NONE;
  }

  void plan_swap_out(int64_t req, int64_t footprint, const int64_t* ext, int64_t n_ext,
                     int64_t tokens) {
    Copy& c = copy_setdefault(req);
    if (!reuse) {
      for (const Seg& s : c.segs)
        if (s.gid != KVC_NONE) pool.free_group(s.gid);
      c.segs.clear();
      drop_prealloc(c);
    }
    int64_t reused = 0;
    std::vector<std::pair<int64_t, int64_t>> holes;
    for (const Seg& s : c.segs) {
      if (!s.valid)
        holes.emplace_back(s.lo, s.hi);
      else if (s.hi <= footprint)
        reused += s.length();
    }
    std::sort(holes.begin(), holes.end());
    const int64_t covered = c.covered();
    const int64_t grow = footprint - covered;
    if (grow > 0) holes.emplace_back(covered, footprint);
    int64_t moved = 0;
    for (auto& h : holes) moved += h.second - h.first;
    const int64_t tail = stale_tail(c, footprint, tokens);

    int64_t absorb = 0;
    if (grow > 0 && c.prealloc != KVC_NONE) absorb = std::min(pool.at(c.prealloc).length, grow);
    try {
      ensure_free(req, moved - absorb);
    } catch (const Err& e) {
      if (e.code != KVC_ERR_CPU_OOM || absorb == 0) throw;
      drop_prealloc(c);  // give the reservation up before failing
      absorb = 0;
      ensure_free(req, moved);
    }

    std::vector<Seg> fresh;
    for (auto& h : holes) {
      int64_t pos = h.first;
      if (h.first == covered && absorb) {
        const int64_t gid = c.prealloc;
        c.prealloc = KVC_NONE;
        pool.shrink_group(gid, absorb);
        fresh.push_back({pos, pos + absorb, gid, true});
        pos += absorb;
      }
      if (pos < h.second) {
        std::vector<Group> grants;
        std::vector<std::pair<int64_t, int64_t>> carved;
        pool.allocate(req, h.second - pos, KVC_NONE, false, grants, carved);
        for (const Group& g : grants) {
          fresh.push_back({pos, pos + g.length, g.id, true});
          pos += g.length;
        }
      }
    }
    std::vector<Seg> segs;
    segs.reserve(c.segs.size() + fresh.size());
    for (const Seg& s : c.segs)
      if (s.valid) segs.push_back(s);
    segs.insert(segs.end(), fresh.begin(), fresh.end());
    std::stable_sort(segs.begin(), segs.end(),
                     [](const Seg& a, const Seg& b) { return a.lo < b.lo; });
    c.segs = std::move(segs);

    const std::vector<Extent> gext = gpu_logical(ext, n_ext);
    std::vector<Extent> fext;
    fext.reserve(fresh.size());
    for (const Seg& s : fresh) fext.push_back({s.lo, s.hi, pool.at(s.gid).start});
    std::vector<Op> ops, refresh;
    pair_extents(holes, gext, fext, ops);  // holes are sorted already
    if (tail != KVC_NONE) {
      const Seg* seg = nullptr;
      for (const Seg& s : c.segs)
        if (s.lo <= tail && tail < s.hi) {
          seg = &s;
          break;
        }
      if (seg == nullptr) fail(KVC_ERR_UNCOVERED, "stale tail block not in the copy");
      if (seg->valid && seg->gid != KVC_NONE && tail < footprint) {
        pair_extents({{tail, tail + 1}}, gext, {{seg->lo, seg->hi, pool.at(seg->gid).start}},
                     refresh);
        ++refreshed;
      }
    }
    if (tokens != KVC_NONE) c.saved = tokens;
    track_peak();
    if (moved + reused != footprint) fail(KVC_ERR_ASSERT, "moved + reused != footprint");
    emit_plan(moved, reused, ops, refresh);
  }

  void emit_plan(int64_t moved, int64_t reused, const std::vector<Op>& ops,
                 const std::vector<Op>& refresh) {
    out.clear();
    out.reserve(4 + 3 * (ops.size() + refresh.size()) + 1);
    out.insert(out.end(), {moved, reused, static_cast<int64_t>(ops.size()),
                           static_cast<int64_t>(refresh.size())});
    for (const Op& o : ops) out.insert(out.end(), {o.blocks, o.gpu, o.cpu});
    for (const Op& o : refresh) out.insert(out.end(), {o.blocks, o.gpu, o.cpu});
  }

  void restore(Copy& c, int64_t blocks, const int64_t* ext, int64_t n_ext) {
    std::vector<std::pair<int64_t, int64_t>> ranges;
    if (blocks) ranges.emplace_back(0, blocks);
    std::vector<Op> ops;
    pair_extents(ranges, gpu_logical(ext, n_ext), host_extents(c), ops);
    emit_plan(blocks, 0, ops, {});
  }

  void plan_swap_in(int64_t req, const int64_t* ext, int64_t n_ext) {
    auto it = copies.find(req);
    if (it == copies.end() || it->second.segs.empty())
      fail(KVC_ERR_CONTAMINATED, "request " + i2s(req) + " has no CPU copy");
    if (!it->second.fully_valid())
      fail(KVC_ERR_CONTAMINATED, "request " + i2s(req) + " copy is contaminated");
    restore(it->second, it->second.covered(), ext, n_ext);
    if (release_on_swap_in) release(req);
  }

  void plan_swap_in_prefix(int64_t req, const int64_t* ext, int64_t n_ext) {
    auto it = copies.find(req);
    if (it == copies.end()) {
      emit_plan(0, 0, {}, {});
      out.push_back(0);
      return;
    }
    Copy& c = it->second;
    const int64_t keep = c.valid_prefix();
    for (const Seg& s : c.segs)
      if (s.lo >= keep && s.gid != KVC_NONE) pool.free_group(s.gid);
    std::vector<Seg> kept;
    for (const Seg& s : c.segs)
      if (s.hi <= keep) kept.push_back(s);
    c.segs = std::move(kept);
    drop_prealloc(c);
    if (c.saved != KVC_NONE) c.saved = std::min(c.saved, keep * block_tokens);
    restore(c, keep, ext, n_ext);
    if (release_on_swap_in) {
      std::vector<int64_t> plan = out;
      release(req);
      out = std::move(plan);
    }
    out.push_back(keep);
  }

  // taken: (owner, gid) pairs, or nullptr
  void evict_for(int64_t rank, int64_t need, std::vector<int64_t>* taken) {
    if (need < 0) fail(KVC_ERR_VALUE, "need_blocks must be >= 0");
    if (need == 0) return;
    std::vector<std::pair<int64_t, Copy*>> victims;  // (owner, copy)
    for (auto& kv : copies)
      if (rank_or0(kv.first) > rank) victims.emplace_back(kv.first, &kv.second);
    std::sort(victims.begin(), victims.end(), [this](const auto& a, const auto& b) {
      const int64_t ra = rank_or0(a.first), rb = rank_or0(b.first);
      return ra != rb ? ra > rb : a.first < b.first;
    });
    int64_t got = 0;
    for (auto& v : victims) {  // reservations hold no data: they go first
      if (got >= need) break;
      got += drop_prealloc(*v.second);
    }
    for (auto& v : victims) {
      if (got >= need) break;
      std::vector<size_t> live;
      for (size_t i = 0; i < v.second->segs.size(); ++i) {
        const Seg& s = v.second->segs[i];
        if (s.valid && s.gid != KVC_NONE) live.push_back(i);
      }
      const std::vector<Seg>& segs = v.second->segs;
      std::stable_sort(live.begin(), live.end(), [&segs](size_t a, size_t b) {
        const int64_t la = segs[a].length(), lb = segs[b].length();
        return la != lb ? la > lb : segs[a].lo < segs[b].lo;
      });
      for (size_t i : live) {
        if (got >= need) break;
        Seg& s = v.second->segs[i];
        const int64_t gid = s.gid;
        got += s.length();
        pool.free_group(gid);
        s.gid = KVC_NONE;
        s.valid = false;
        if (taken) taken->insert(taken->end(), {v.first, gid});
      }
    }
    if (got < need)
      fail(KVC_ERR_INSUFFICIENT, "only " + i2s(got) + " of " + i2s(need) +
                                     " blocks evictable below rank " + i2s(rank));
  }

  bool preallocate_increment(int64_t req, int64_t inc) {
    if (inc == 0) return true;
    auto it = copies.find(req);
    if (it == copies.end() || it->second.segs.empty() || !it->second.fully_valid()) return false;
    Copy& c = it->second;
    if (c.prealloc != KVC_NONE) return true;
    const int64_t after = pool.at(c.segs.back().gid).end();
    Group g{};
    if (!pool.allocate_at(req, after, inc, &g)) return false;
    c.prealloc = g.id;
    track_peak();
    return true;
  }

  void release(int64_t req) {
    auto it = copies.find(req);
    if (it == copies.end()) return;
    Copy c = std::move(it->second);
    copies.erase(it);
    for (const Seg& s : c.segs)
      if (s.gid != KVC_NONE) pool.free_group(s.gid);
    c.segs.clear();
    drop_prealloc(c);
    ranks.erase(req);
  }
};

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
namespace kvc {

template <typename F>
int guard(F&& f) {
  try {
    f();
    return KVC_OK;
  } catch (const Err& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "out of host memory";
    return KVC_ERR_POOL;
  }
}

void give_out(std::vector<int64_t>& v, const int64_t** res, int64_t* len) {
  *res = v.data();
  *len = static_cast<int64_t>(v.size());
}

void check_ptr(const void* p) {
  if (p == nullptr) fail(KVC_ERR_VALUE, "null handle or output pointer");
}

}  // namespace kvc

extern "C" {

int kvc_abi_version(void) { return KVC_ABI_VERSION; }
const char* kvc_last_error(void) { return g_err.c_str(); }

int kvc_rng_draws(const int64_t* entropy, int32_t n_entropy, int64_t bound, int64_t n,
                  int64_t* out) {
  return guard([&] {
    check_ptr(out);
    if (n_entropy < 0 || (n_entropy > 0 && entropy == nullptr)) fail(KVC_ERR_VALUE, "entropy");
    Pcg64 r;
    r.seed(coerce_entropy(entropy, n_entropy));
    for (int64_t i = 0; i < n; ++i) out[i] = r.integers(bound);
  });
}

int kvc_pool_create(int64_t total_blocks, int64_t initial_group_blocks, int64_t rng_seed,
                    int victim_policy, KvcPool** out) {
  return guard([&] {
    check_ptr(out);
    if (total_blocks < 1)
      fail(KVC_ERR_VALUE, "total_blocks must be >= 1, got " + i2s(total_blocks));
    if (initial_group_blocks < 1)
      fail(KVC_ERR_VALUE,
           "initial_group_blocks must be >= 1, got " + i2s(initial_group_blocks));
    if (initial_group_blocks > total_blocks)
      fail(KVC_ERR_VALUE, "total_blocks must be >= initial_group_blocks");
    if (victim_policy != KVC_VICTIM_RANDOM && victim_policy != KVC_VICTIM_LOWEST_PRIORITY)
      fail(KVC_ERR_VALUE, "unknown victim_policy");
    auto* p = new KvcPool();
    p->total = total_blocks;
    p->initial = initial_group_blocks;
    p->victim_policy = victim_policy;
    const int64_t entropy[2] = {rng_seed, kAllocRngLabel};
    try {
      p->rng.seed(coerce_entropy(entropy, 2));
    } catch (...) {
      delete p;
      throw;
    }
    p->free_total = total_blocks;
    p->link(p->fresh(0, total_blocks, true));
    *out = p;
  });
}

int kvc_pool_destroy(KvcPool* p) {
  delete p;
  return KVC_OK;
}

int kvc_pool_set_rank_fn(KvcPool* p, kvc_rank_fn fn, void* ctx) {
  return guard([&] {
    check_ptr(p);
    p->rank_fn = fn;
    p->rank_ctx = ctx;
  });
}

int kvc_pool_allocate(KvcPool* p, int64_t req, int64_t want, int64_t expected_total,
                      int reclaim, const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(p);
    std::vector<Group> grants;
    std::vector<std::pair<int64_t, int64_t>> carved;
    p->allocate(req, want, expected_total, reclaim != 0, grants, carved);
    p->out.clear();
    p->out.push_back(static_cast<int64_t>(grants.size()));
    p->out.push_back(static_cast<int64_t>(carved.size()));
    for (const Group& g : grants) p->out.insert(p->out.end(), {g.id, g.start, g.length});
    for (auto& c : carved) p->out.insert(p->out.end(), {c.first, c.second});
    give_out(p->out, res, len);
  });
}

int kvc_pool_reclaim_from_victim(KvcPool* p, int64_t need, int64_t for_request,
                                 const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(p);
    auto r = p->reclaim_from_victim(need, for_request);
    p->out.assign({r.first, r.second.id, r.second.start, r.second.length});
    give_out(p->out, res, len);
  });
}

int kvc_pool_allocate_at(KvcPool* p, int64_t req, int64_t start, int64_t length,
                         const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(p);
    Group g{};
    p->out.clear();
    if (p->allocate_at(req, start, length, &g)) p->out.assign({g.id, g.start, g.length});
    give_out(p->out, res, len);
  });
}

int kvc_pool_free_group(KvcPool* p, int64_t gid) {
  return guard([&] {
    check_ptr(p);
    p->free_group(gid);
  });
}

int kvc_pool_shrink_group(KvcPool* p, int64_t gid, int64_t new_length) {
  return guard([&] {
    check_ptr(p);
    p->shrink_group(gid, new_length);
  });
}

int kvc_pool_free_request(KvcPool* p, int64_t req, int64_t* freed) {
  return guard([&] {
    check_ptr(p);
    check_ptr(freed);
    *freed = p->free_request(req);
  });
}

int kvc_pool_set_request_fill(KvcPool* p, int64_t req, int64_t filled_blocks) {
  return guard([&] {
    check_ptr(p);
    p->set_request_fill(req, filled_blocks);
  });
}

int kvc_pool_record_transfer(KvcPool* p, int64_t blocks) {
  return guard([&] {
    check_ptr(p);
    p->sizes[blocks] += 1;
    p->ops_recorded += 1;
    p->blocks_recorded += blocks;
  });
}

int kvc_pool_counters(KvcPool* p, int64_t* out6) {
  return guard([&] {
    check_ptr(p);
    check_ptr(out6);
    out6[0] = p->total;
    out6[1] = p->free_total;
    out6[2] = p->total - p->free_total;
    out6[3] = static_cast<int64_t>(p->groups.size());
    out6[4] = p->ops_recorded;
    out6[5] = p->blocks_recorded;
  });
}

int kvc_pool_owned_blocks(KvcPool* p, int64_t req, int64_t* out) {
  return guard([&] {
    check_ptr(p);
    check_ptr(out);
    *out = p->owned_blocks(req);
  });
}

int kvc_pool_reclaimable_blocks(KvcPool* p, int64_t exclude, int64_t* out) {
  return guard([&] {
    check_ptr(p);
    check_ptr(out);
    *out = p->reclaimable(exclude);
  });
}

int kvc_pool_group(KvcPool* p, int64_t gid, int64_t* out7) {
  return guard([&] {
    check_ptr(p);
    check_ptr(out7);
    const Group& g = p->at(gid);
    const int64_t v[7] = {g.id, g.start, g.length, g.free ? 1 : 0, g.owner, g.active ? 1 : 0,
                          g.filled};
    std::memcpy(out7, v, sizeof v);
  });
}

int kvc_pool_owned_groups(KvcPool* p, int64_t req, const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(p);
    p->out.clear();
    auto it = p->owned.find(req);
    if (it != p->owned.end())
      for (int64_t gid : it->second) p->put(p->groups.at(gid));
    give_out(p->out, res, len);
  });
}

int kvc_pool_free_groups(KvcPool* p, const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(p);
    p->out.clear();
    for (auto& a : p->by_addr) p->put(p->groups.at(a.second));
    give_out(p->out, res, len);
  });
}

int kvc_pool_extents(KvcPool* p, int64_t req, const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(p);
    p->out.clear();
    auto it = p->owned.find(req);
    if (it != p->owned.end())
      for (int64_t gid : it->second) {
        const Group& g = p->groups.at(gid);
        const size_t n = p->out.size();
        if (n >= 2 && p->out[n - 2] + p->out[n - 1] == g.start)
          p->out[n - 1] += g.length;
        else
          p->out.insert(p->out.end(), {g.start, g.length});
      }
    give_out(p->out, res, len);
  });
}

int kvc_pool_set_group_filled(KvcPool* p, int64_t gid, int64_t filled) {
  return guard([&] {
    check_ptr(p);
    p->at(gid).filled = filled;
  });
}

int kvc_pool_granularity(KvcPool* p, const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(p);
    p->out.clear();
    for (auto& kv : p->sizes) p->out.insert(p->out.end(), {kv.first, kv.second});
    give_out(p->out, res, len);
  });
}

int kvc_pool_dump(KvcPool* p, char* buf, int64_t cap, int64_t* need) {
  return guard([&] {
    check_ptr(p);
    check_ptr(need);
    p->text = p->dump();
    *need = static_cast<int64_t>(p->text.size()) + 1;
    if (buf != nullptr && cap >= *need) std::memcpy(buf, p->text.c_str(), p->text.size() + 1);
  });
}

int kvc_pool_validate(KvcPool* p) {
  return guard([&] {
    check_ptr(p);
    p->validate();
  });
}

int kvc_store_create(int64_t total_blocks, int reuse_enabled, int64_t prealloc_min_blocks,
                     int64_t prealloc_max_blocks, int release_on_swap_in,
                     int64_t block_size_tokens, KvcStore** out) {
  return guard([&] {
    check_ptr(out);
    if (total_blocks < 1)
      fail(KVC_ERR_VALUE, "total_blocks must be >= 1, got " + i2s(total_blocks));
    if (block_size_tokens < 1) fail(KVC_ERR_VALUE, "block_size_tokens must be >= 1");
    auto* s = new KvcStore();
    s->pool.total = total_blocks;
    s->pool.initial = 1;  // cpu_store.py:134
    const int64_t entropy[2] = {0, kAllocRngLabel};
    s->pool.rng.seed(coerce_entropy(entropy, 2));
    s->pool.free_total = total_blocks;
    s->pool.link(s->pool.fresh(0, total_blocks, true));
    s->reuse = reuse_enabled != 0;
    s->pmin = prealloc_min_blocks;
    s->pmax = prealloc_max_blocks;
    s->release_on_swap_in = release_on_swap_in != 0;
    s->block_tokens = block_size_tokens;
    *out = s;
  });
}

int kvc_store_destroy(KvcStore* s) {
  delete s;
  return KVC_OK;
}

int kvc_store_pool(KvcStore* s, KvcPool** out) {
  return guard([&] {
    check_ptr(s);
    check_ptr(out);
    *out = &s->pool;
  });
}

int kvc_store_set_flag(KvcStore* s, int which, int64_t value) {
  return guard([&] {
    check_ptr(s);
    switch (which) {
      case 0: s->reuse = value != 0; break;
      case 1: s->refresh_dirty_tail = value != 0; break;
      case 2: s->release_on_swap_in = value != 0; break;
      default: fail(KVC_ERR_VALUE, "unknown store flag " + i2s(which));
    }
  });
}

int kvc_store_counters(KvcStore* s, int64_t* out5) {
  return guard([&] {
    check_ptr(s);
    check_ptr(out5);
    out5[0] = s->peak;
    out5[1] = s->refreshed;
    out5[2] = static_cast<int64_t>(s->copies.size());
    out5[3] = static_cast<int64_t>(s->ranks.size());
    out5[4] = s->refresh_dirty_tail ? 1 : 0;
  });
}

int kvc_store_set_rank(KvcStore* s, int64_t req, int64_t rank) {
  return guard([&] {
    check_ptr(s);
    s->ranks[req] = rank;
  });
}

int kvc_store_set_ranks(KvcStore* s, const int64_t* pairs, int64_t n) {
  return guard([&] {
    check_ptr(s);
    if (n < 0 || (n > 0 && pairs == nullptr)) fail(KVC_ERR_VALUE, "rank pairs");
    for (int64_t i = 0; i < n; ++i) s->ranks[pairs[2 * i]] = pairs[2 * i + 1];
  });
}

int kvc_store_ensure_free(KvcStore* s, int64_t req, int64_t need) {
  return guard([&] {
    check_ptr(s);
    s->ensure_free(req, need);
  });
}

int kvc_store_track_peak(KvcStore* s) {
  return guard([&] {
    check_ptr(s);
    s->track_peak();
  });
}

int kvc_store_get_rank(KvcStore* s, int64_t req, int64_t* rank) {
  return guard([&] {
    check_ptr(s);
    check_ptr(rank);
    auto it = s->ranks.find(req);
    *rank = it == s->ranks.end() ? KVC_NONE : it->second;
  });
}

int kvc_store_del_rank(KvcStore* s, int64_t req) {
  return guard([&] {
    check_ptr(s);
    if (s->ranks.erase(req) == 0) fail(KVC_ERR_KEY, i2s(req));
  });
}

int kvc_store_ranks(KvcStore* s, const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(s);
    s->out.clear();
    for (auto& kv : s->ranks) s->out.insert(s->out.end(), {kv.first, kv.second});
    give_out(s->out, res, len);
  });
}

int kvc_store_clear_ranks(KvcStore* s) {
  return guard([&] {
    check_ptr(s);
    s->ranks.clear();
  });
}

int kvc_store_plan_swap_out(KvcStore* s, int64_t req, int64_t footprint, const int64_t* extents,
                            int64_t n_extents, int64_t tokens, const int64_t** res,
                            int64_t* len) {
  return guard([&] {
    check_ptr(s);
    if (n_extents < 0 || (n_extents > 0 && extents == nullptr)) fail(KVC_ERR_VALUE, "extents");
    s->plan_swap_out(req, footprint, extents, n_extents, tokens);
    give_out(s->out, res, len);
  });
}

int kvc_store_plan_swap_in(KvcStore* s, int64_t req, const int64_t* extents, int64_t n_extents,
                           const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(s);
    if (n_extents < 0 || (n_extents > 0 && extents == nullptr)) fail(KVC_ERR_VALUE, "extents");
    s->plan_swap_in(req, extents, n_extents);
    give_out(s->out, res, len);
  });
}

int kvc_store_plan_swap_in_prefix(KvcStore* s, int64_t req, const int64_t* extents,
                                  int64_t n_extents, const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(s);
    if (n_extents < 0 || (n_extents > 0 && extents == nullptr)) fail(KVC_ERR_VALUE, "extents");
    s->plan_swap_in_prefix(req, extents, n_extents);
    give_out(s->out, res, len);
  });
}

int kvc_store_evict_for(KvcStore* s, int64_t rank, int64_t need, const int64_t** res,
                        int64_t* len) {
  return guard([&] {
    check_ptr(s);
    s->out.clear();
    std::vector<int64_t> taken;
    s->evict_for(rank, need, &taken);
    s->out = std::move(taken);
    give_out(s->out, res, len);
  });
}

int kvc_store_preallocate_increment(KvcStore* s, int64_t req, int64_t expected_increment,
                                    int* ok) {
  return guard([&] {
    check_ptr(s);
    check_ptr(ok);
    *ok = s->preallocate_increment(req, expected_increment) ? 1 : 0;
  });
}

int kvc_store_release(KvcStore* s, int64_t req) {
  return guard([&] {
    check_ptr(s);
    s->release(req);
  });
}

int kvc_store_copy_ids(KvcStore* s, const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(s);
    std::vector<std::pair<int64_t, int64_t>> order;
    for (auto& kv : s->copies) order.emplace_back(kv.second.order, kv.first);
    std::sort(order.begin(), order.end());
    s->out.clear();
    for (auto& o : order) s->out.push_back(o.second);
    give_out(s->out, res, len);
  });
}

int kvc_store_copy(KvcStore* s, int64_t req, const int64_t** res, int64_t* len) {
  return guard([&] {
    check_ptr(s);
    auto it = s->copies.find(req);
    if (it == s->copies.end()) fail(KVC_ERR_KEY, i2s(req));
    const Copy& c = it->second;
    s->out.assign({c.prealloc, c.saved, static_cast<int64_t>(c.segs.size())});
    for (const Seg& g : c.segs) s->out.insert(s->out.end(), {g.lo, g.hi, g.gid, g.valid ? 1 : 0});
    give_out(s->out, res, len);
  });
}

int kvc_store_put_copy(KvcStore* s, int64_t req, int64_t prealloc, int64_t saved_tokens,
                       const int64_t* segs, int64_t n_segs) {
  return guard([&] {
    check_ptr(s);
    if (n_segs < 0 || (n_segs > 0 && segs == nullptr)) fail(KVC_ERR_VALUE, "segments");
    Copy& c = s->copy_setdefault(req);
    c.prealloc = prealloc;
    c.saved = saved_tokens;
    c.segs.clear();
    for (int64_t i = 0; i < n_segs; ++i)
      c.segs.push_back({segs[4 * i], segs[4 * i + 1], segs[4 * i + 2], segs[4 * i + 3] != 0});
  });
}

int kvc_store_drop_copy(KvcStore* s, int64_t req) {
  return guard([&] {
    check_ptr(s);
    if (s->copies.erase(req) == 0) fail(KVC_ERR_KEY, i2s(req));
  });
}

}  // extern "C"
