// abi.cu -- the C ABI (include/smgpu.h): argument checking, planning (order pi,
// peeling factor r, strategy, tiling) and launch orchestration.  Host code only;
// every step of the path on the text runs in the kernels of this library.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "launch.h"
#include "smgpu.h"

using namespace smgpu;

namespace {

thread_local sm_status g_status = SM_OK;
thread_local std::string g_message;
thread_local uint64_t g_launches = 0;

sm_status fail(sm_status s, const std::string& msg) {
  g_status = s;
  g_message = msg;
  return s;
}

sm_status cuda_fail(cudaError_t e, const char* what) {
  std::string msg = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return fail(e == cudaErrorMemoryAllocation ? SM_ENOMEM : SM_ECUDA, msg);
}

#define SM_CUDA_TRY(expr, what)                      \
  do {                                               \
    cudaError_t _e = (expr);                         \
    if (_e != cudaSuccess) return cuda_fail(_e, what); \
  } while (0)

#ifdef SMGPU_COUNTERS
// instrumented build: one device u64[kCounters] per device, accumulated by every launch
unsigned long long* counters_ptr() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  static unsigned long long* bufs[64] = {nullptr};
  if (!bufs[dev]) {
    void* q = nullptr;
    if (cudaMalloc(&q, kCounters * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
    cudaMemset(q, 0, kCounters * sizeof(unsigned long long));
    bufs[dev] = static_cast<unsigned long long*>(q);
  }
  return bufs[dev];
}
#else
unsigned long long* counters_ptr() { return nullptr; }
#endif

int num_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  static int cache[64] = {0};
  if (dev < 64 && cache[dev]) return cache[dev];
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (dev < 64) cache[dev] = sms;
  return sms;
}

cudaStream_t as_stream(void* s) { return s ? reinterpret_cast<cudaStream_t>(s) : cudaStreamPerThread; }

sm_status check_device_ptr(const void* ptr, const char* name) {
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, ptr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(SM_EINVAL, std::string(name) + " is not a CUDA-visible pointer");
  }
  if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged)
    return fail(SM_EINVAL, std::string(name) + " must be device memory (no CPU fallback)");
  int dev = 0;
  cudaGetDevice(&dev);
  if (at.type == cudaMemoryTypeDevice && at.device != dev)
    return fail(SM_EINVAL, std::string(name) + " lives on another device than the current one");
  return SM_OK;
}

sm_status check_pattern_text(const uint8_t* p, size_t m, const uint8_t* t, size_t n) {
  if (m == 0) return fail(SM_EINVAL, "m == 0: empty pattern is undefined (reading R2)");
  if (m > SM_MAX_PATTERN) return fail(SM_EINVAL, "m > SM_MAX_PATTERN (4096)");
  if (!p) return fail(SM_EINVAL, "p is NULL");
  if (n > 0) {
    if (!t) return fail(SM_EINVAL, "t is NULL with n > 0");
    sm_status s = check_device_ptr(t, "t");
    if (s != SM_OK) return s;
  }
  return SM_OK;
}

// stable rarest-first order (ties by position, R11).  A stable
// counting sort: the distinct key values hist[c] of the symbols in p are ranked
// (at most 256 of them), then positions are bucketed by rank in ascending order
// (stable: ascending position within a bucket).  O(m + sigma_p^2) for sigma_p distinct
// symbols in p; equals std::stable_sort by hist[p[j]].
void order_from_hist(const uint64_t* hist, const uint8_t* p, size_t m, uint32_t* order) {
  // distinct symbols of p in first-occurrence order (a pattern holds few: 4 for DNA)
  uint8_t slot[256];
  uint64_t seen[4] = {0, 0, 0, 0};
  uint8_t syms[256];
  int ns = 0;
  for (size_t j = 0; j < m; ++j) {
    const uint8_t c = p[j];
    if (!(seen[c >> 6] >> (c & 63) & 1u)) {
      seen[c >> 6] |= 1ull << (c & 63);
      syms[ns++] = c;
    }
  }
  // rank the distinct count values: insertion sort of the symbols by hist (ns is small)
  for (int i = 1; i < ns; ++i) {
    const uint8_t c = syms[i];
    const uint64_t key = hist[c];
    int k = i;
    while (k > 0 && hist[syms[k - 1]] > key) {
      syms[k] = syms[k - 1];
      --k;
    }
    syms[k] = c;
  }
  uint32_t start[257];
  int nr = 0;
  for (int i = 0; i < ns; ++i) {
    if (i > 0 && hist[syms[i]] != hist[syms[i - 1]]) ++nr;
    slot[syms[i]] = (uint8_t)nr;
  }
  ++nr;
  for (int r = 0; r <= nr; ++r) start[r] = 0;
  for (size_t j = 0; j < m; ++j) ++start[slot[p[j]] + 1];
  for (int r = 0; r < nr; ++r) start[r + 1] += start[r];
  for (size_t j = 0; j < m; ++j) order[start[slot[p[j]]]++] = (uint32_t)j;
}

bool valid_permutation(const uint32_t* order, size_t m) {
  std::vector<char> seen(m, 0);
  for (size_t k = 0; k < m; ++k) {
    if (order[k] >= m || seen[order[k]]) return false;
    seen[order[k]] = 1;
  }
  return true;
}

// Performance knobs (never change results).  Defaults tuned on B200; SMGPU_* env
// variables override them once per process for tuning sweeps.
struct Tunables {
  uint32_t tile = 32768;        // text bytes per tile for large texts (4096 * CPL)
  int ctas_per_sm = 3;          // persistent CTAs per SM (3 x 2 stages beat 2 x 3 stages by ~11 %: more
                                // resident warps; the planner falls back to 2 when 2 stages do not fit)
  uint32_t max_stages = 8;      // ring depth cap per CTA
  bool auto_packed = true;      // AUTO may pick PACKED for small text alphabets
  bool alternate = true;        // batches: odd patterns scan the text backwards (L2 reuse at the seam)
  double pair_min_hit = 0.2;    // AUTO: PAIR instead of FILTER when p[pi(1)] is in > this share of 16-B chunks
  double pair_min_hit_long = 0.12;  // ... for m >= 32 (a word-aligned pi(2) is then almost always available)
  double block_min_hit = 0.5;   // AUTO: BLOCK / PACKED when a pi(1)&pi(2) survivor is in > this share
  uint32_t l2_policy = 0;       // TMA load L2 policy: 0 evict_first, 1 evict_normal, 2 evict_last
  bool prepack = true;          // batches over <= 4-symbol texts: pack the text once (NEXT-3)
  uint32_t prepack_min_p = 2;   // ... when the call has at least this many patterns
  double pair_align_slack = 6;  // PAIR: prefer a word-aligned pi(2) within this frequency factor (<= 1: off)
  int peel_bias = 0;            // added to the AUTO peeling factor (tuning; +2 measured slower)
  uint32_t wait_ns = 0;         // consumers' stage wait: suspend-time hint in ns (0 = spin)
  int ctas_pre = 3;             // persistent CTAs per SM for the pre-packed PACKED kernels (small stages)
  uint32_t max_stages_pre = 6;  // their ring depth (3 CTAs x 6 stages of <= 9 KiB fit the SM)
  bool dispatch = true;         // batch calls: work items fetched from a counter (search.cuh work_ctr)
  uint64_t dispatch_min_bytes = 64ull << 20;  // ... when the call streams at least this much text (n x P)
  uint64_t dispatch_min_bytes_single = 512ull << 20;  // single-pattern calls (the counter's memset
                                                      // costs more than it gains on short launches)
  uint32_t list_max = 65535;    // reporting: a warp stages a u16 list for <= this many matches, else its bitmap
};

const Tunables& tunables() {
  static const Tunables t = [] {
    Tunables x;
    if (const char* e = std::getenv("SMGPU_TILE")) x.tile = (uint32_t)std::atoi(e);
    if (const char* e = std::getenv("SMGPU_CTAS_PER_SM")) x.ctas_per_sm = std::atoi(e);
    if (const char* e = std::getenv("SMGPU_STAGES")) x.max_stages = (uint32_t)std::atoi(e);
    if (const char* e = std::getenv("SMGPU_AUTO_PACKED")) x.auto_packed = std::atoi(e) != 0;
    if (const char* e = std::getenv("SMGPU_ALTERNATE")) x.alternate = std::atoi(e) != 0;
    if (const char* e = std::getenv("SMGPU_PAIR_MIN_HIT")) x.pair_min_hit = std::atof(e);
    if (const char* e = std::getenv("SMGPU_PAIR_MIN_HIT_LONG")) x.pair_min_hit_long = std::atof(e);
    if (const char* e = std::getenv("SMGPU_BLOCK_MIN_HIT")) x.block_min_hit = std::atof(e);
    if (const char* e = std::getenv("SMGPU_L2_POLICY")) x.l2_policy = (uint32_t)std::atoi(e) % 3u;
    if (const char* e = std::getenv("SMGPU_PREPACK")) x.prepack = std::atoi(e) != 0;
    if (const char* e = std::getenv("SMGPU_PREPACK_MIN_P")) x.prepack_min_p = (uint32_t)std::atoi(e);
    if (const char* e = std::getenv("SMGPU_PAIR_ALIGN")) x.pair_align_slack = std::atof(e);
    if (const char* e = std::getenv("SMGPU_PEEL_BIAS")) x.peel_bias = std::atoi(e);
    if (const char* e = std::getenv("SMGPU_WAIT_NS")) x.wait_ns = (uint32_t)std::atoi(e);
    if (const char* e = std::getenv("SMGPU_CTAS_PRE")) x.ctas_pre = std::atoi(e);
    if (const char* e = std::getenv("SMGPU_DISPATCH")) x.dispatch = std::atoi(e) != 0;
    if (const char* e = std::getenv("SMGPU_DISPATCH_MIN_MB")) x.dispatch_min_bytes = (uint64_t)std::atoll(e) << 20;
    if (const char* e = std::getenv("SMGPU_DISPATCH_MIN_MB_SINGLE"))
      x.dispatch_min_bytes_single = (uint64_t)std::atoll(e) << 20;
    if (const char* e = std::getenv("SMGPU_LIST_MAX")) x.list_max = (uint32_t)std::atoi(e);
    if (x.ctas_pre < 1 || x.ctas_pre > 4) x.ctas_pre = 3;
    if (const char* e = std::getenv("SMGPU_STAGES_PRE")) x.max_stages_pre = (uint32_t)std::atoi(e);
    if (x.max_stages_pre < 2 || x.max_stages_pre > (uint32_t)kMaxStages) x.max_stages_pre = 6;
    if (x.tile != 4096 && x.tile != 8192 && x.tile != 16384 && x.tile != 32768) x.tile = 32768;
    if (x.ctas_per_sm < 1 || x.ctas_per_sm > 4) x.ctas_per_sm = 3;
    if (x.max_stages < 2 || x.max_stages > (uint32_t)kMaxStages) x.max_stages = kMaxStages;
    return x;
  }();
  return t;
}

// counter-dispatched work items (search.cuh work_ctr) for calls streaming enough text
bool use_dispatch(uint64_t n, size_t P) {
  const Tunables& tu = tunables();
  return tu.dispatch && n * P >= (P == 1 ? tu.dispatch_min_bytes_single : tu.dispatch_min_bytes);
}

// The comparison order of one plan: inline for m <= 64 (no allocation per pattern on
// the planning path of a batch call), on the heap beyond.
class OrderVec {
 public:
  void resize(size_t m) {
    m_ = m;
    if (m > kInline) heap_.resize(m);
  }
  size_t size() const { return m_; }
  uint32_t* data() { return m_ > kInline ? heap_.data() : small_; }
  const uint32_t* data() const { return m_ > kInline ? heap_.data() : small_; }
  uint32_t& operator[](size_t k) { return data()[k]; }
  const uint32_t& operator[](size_t k) const { return data()[k]; }

 private:
  static constexpr size_t kInline = 64;
  size_t m_ = 0;
  uint32_t small_[kInline];
  std::vector<uint32_t> heap_;
};

struct Plan {
  int strategy = kFilter;
  uint32_t code_shift = 0;  // PACKED: code field shift
  uint32_t r = 1;
  int cpl = 4;
  uint32_t tile = 16384;
  OrderVec order;
};


// P = patterns of the call: a launch holds up to kMaxBatch of them, each a full pass,
// so its work items are tiles x min(P, kMaxBatch)
void choose_tiling(uint64_t n, size_t P, Plan& pl) {
  const uint64_t sms = (uint64_t)num_sms();
  const uint64_t per_launch = std::max<uint64_t>(1, std::min<uint64_t>(P, kMaxBatch));
  pl.tile = tunables().tile;
  // small texts: shrink the tile until every CTA slot gets work
  while (pl.tile > 4096 && (n + pl.tile - 1) / pl.tile * per_launch < sms * (uint64_t)tunables().ctas_per_sm)
    pl.tile /= 2;
  pl.cpl = (int)(pl.tile / (16u * kLanesPerTilePass));
}

// PACKED applicability: a b-bit field (x >> s) & (2^b - 1), b in {1, 2}, that is
// injective on the symbols present in t, and every pattern symbol present in t.
// Returns the strategy (kPacked1 / kPacked2) or 0; *shift receives s.
// The b-bit code field of the text (b in {1, 2}): (x >> s) & (2^b - 1) injective on the
// symbols present in t.  Returns b (0 if none) and *shift = s.
int text_code_bits(const uint64_t* hist, uint32_t* shift) {
  int present = 0;
  for (int c = 0; c < 256; ++c) present += hist[c] > 0;
  for (int b = 1; b <= 2; ++b) {
    if (present > (1 << b)) continue;
    for (uint32_t s = 0; s + b <= 8; ++s) {
      bool used[4] = {false, false, false, false};
      bool ok = true;
      for (int c = 0; c < 256 && ok; ++c) {
        if (!hist[c]) continue;
        const uint32_t code = ((uint32_t)c >> s) & ((1u << b) - 1u);
        if (used[code]) ok = false;
        used[code] = true;
      }
      if (ok) {
        *shift = s;
        return b;
      }
    }
  }
  return 0;
}


// Per-call scratch (report staging, code arrays, count cells) comes from the library's
// own stream-ordered pool per device -- not the device's default pool, whose attributes
// belong to the process.  Freed blocks stay cached across synchronisations up to
// SMGPU_POOL_KEEP_BYTES (default: all), so repeated calls cost no remapping (a 1 GiB cap
// cost 12.5 ms per c2 report call: its 2-4 GiB staging pool was unmapped and remapped
// every call, profiles/report_r2.md); sm_trim_scratch() hands the cached memory back.
uint64_t pool_keep_bytes() {
  static const uint64_t v = [] {
    const char* e = std::getenv("SMGPU_POOL_KEEP_BYTES");
    return e ? (uint64_t)std::strtoull(e, nullptr, 10) : UINT64_MAX;
  }();
  return v;
}

cudaMemPool_t g_pools[64] = {};
std::mutex g_pool_mu;

cudaError_t pool_alloc(void** ptr, size_t bytes, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaMallocAsync(ptr, bytes, st);
  cudaMemPool_t pool;
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    cudaMemPool_t* pools = g_pools;
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.handleTypes = cudaMemHandleTypeNone;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      cudaMemPool_t p;
      e = cudaMemPoolCreate(&p, &props);
      if (e != cudaSuccess) return e;
      uint64_t thr = pool_keep_bytes();
      cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
      pools[dev] = p;
    }
    pool = pools[dev];
  }
  return cudaMallocFromPoolAsync(ptr, bytes, pool, st);
}

// NEXT-3: for a batch of >= 2 patterns over a <= 4-symbol text, pack the text once
// into its code array and run the PACKED patterns on it (kPackedBPre).  Returns the
// array (stream-ordered allocation, caller frees) or nullptr; *b_out = code bits.
// guard (hist is the caller's, not computed here from t -- PAPER.md:113 allows corpus
// frequencies, which need not be t's): packs for any P, and the pack kernel also checks
// that every text byte is one of the symbols the code field was chosen for, setting the
// device flag *flag_out (u32 after the array) otherwise.  The PACKED launches on the
// array then run guarded (kGuardClear) next to a byte-compare fallback (kGuardSet), so
// a histogram that is not t's can change the speed but never the result.
uint8_t* prepack_text(const uint64_t* hist, const uint8_t* t, size_t n, size_t P, bool guard, cudaStream_t st,
                      int* b_out, uint32_t** flag_out, cudaError_t* err) {
  *err = cudaSuccess;
  *b_out = 0;
  *flag_out = nullptr;
  if (!tunables().prepack || (!guard && P < std::max<uint32_t>(1u, tunables().prepack_min_p)) || n == 0 || P == 0)
    return nullptr;
  uint32_t shift = 0;
  const int b = text_code_bits(hist, &shift);
  if (!b) return nullptr;
  uint32_t syms = 0;  // the (<= 4) symbols present per hist, the first repeated to fill 4 bytes
  int ns = 0;
  for (int c = 0; c < 256; ++c)
    if (hist[c]) syms |= (uint32_t)c << (8 * ns++);
  for (int i = ns; i < 4; ++i) syms |= (syms & 0xFFu) << (8 * i);
  const uintptr_t tp = reinterpret_cast<uintptr_t>(t);
  const uint64_t delta = tp & 15;
  // alignments covered: every tile of every pattern plus the largest post region
  const uint64_t X = ((delta + n + 32767) / 32768 + 1) * 32768 + 8192;
  const uint64_t bytes = ((X * (uint64_t)b / 8) + 15) & ~15ull;
  uint8_t* codes = nullptr;
  *err = pool_alloc(reinterpret_cast<void**>(&codes), bytes + (guard ? 16 : 0), st);
  if (*err != cudaSuccess) return nullptr;
  uint32_t* flag = guard ? reinterpret_cast<uint32_t*>(codes + bytes) : nullptr;
  if (flag) *err = cudaMemsetAsync(flag, 0, 4, st);
  if (*err == cudaSuccess)
    *err = launch_pack_text(reinterpret_cast<const uint8_t*>(tp & ~(uintptr_t)15), delta, n, shift, b, codes, bytes,
                            syms, flag, num_sms(), st);
  if (*err != cudaSuccess) {
    cudaFreeAsync(codes, st);
    return nullptr;
  }
  ++g_launches;
  *b_out = b;
  *flag_out = flag;
  return codes;
}

// the pre-packed code array of one batch call (freed stream-ordered at scope end)
struct CodeArray {
  uint8_t* p;
  cudaStream_t st;
  ~CodeArray() {
    if (p) cudaFreeAsync(p, st);
  }
};

// a PACKED plan runs on the batch's code array when there is one (same b: same text)
void use_codes(const CodeArray& codes, int cb, Plan& pl) {
  if (codes.p && is_packed(pl.strategy) && !is_prepacked(pl.strategy) && code_bits(pl.strategy) == cb)
    pl.strategy += kPacked1Pre - kPacked1;
}

// Per-text facts every plan of a call needs (computed once per call, not per pattern).
struct TextInfo {
  double total = 0;         // n from the histogram
  int code_b = 0;           // text_code_bits: 0, 1 or 2
  uint32_t code_shift = 0;
  Plan tiling;              // choose_tiling(n, P): tile and CPL
};

TextInfo text_info(const uint64_t* hist, uint64_t n, size_t P = 1) {
  TextInfo t;
  for (int c = 0; c < 256; ++c) t.total += (double)hist[c];
  t.code_b = text_code_bits(hist, &t.code_shift);
  choose_tiling(n, P, t.tiling);
  return t;
}

// allow_packed = false: PACKED is never chosen (AUTO keeps the byte strategy; a forced
// SM_STRATEGY_PACKED runs BLOCK, the same comparisons on bytes) -- for a caller histogram
// whose code field the device cannot check, and for the guarded fallback launches.
sm_status make_plan(const uint8_t* p, size_t m, uint64_t n, const uint64_t* hist, const uint32_t* order,
                    uint32_t peel, int strategy, Plan& pl, const TextInfo* tinfo = nullptr,
                    bool allow_packed = true) {
  if (strategy < SM_STRATEGY_AUTO || strategy > SM_STRATEGY_PAIR) return fail(SM_EINVAL, "bad strategy");
  TextInfo local;
  if (!tinfo) {
    local = text_info(hist, n);
    tinfo = &local;
  }
  // PACKED applicability: the text's code field and every pattern symbol present in t
  auto packed = [&]() -> int {
    for (size_t j = 0; j < m; ++j)
      if (hist[p[j]] == 0) return 0;  // an absent symbol: FILTER answers 0 at once
    pl.code_shift = tinfo->code_shift;
    return tinfo->code_b == 1 ? kPacked1 : (tinfo->code_b == 2 ? kPacked2 : 0);
  };
  pl.order.resize(m);
  if (order) {
    if (!valid_permutation(order, m)) return fail(SM_EINVAL, "order is not a permutation of 0..m-1");
    std::memcpy(pl.order.data(), order, m * sizeof(uint32_t));
  } else {
    order_from_hist(hist, p, m, pl.order.data());
  }
  pl.tile = tinfo->tiling.tile;
  pl.cpl = tinfo->tiling.cpl;
  const double total = tinfo->total;
  auto freq = [&](size_t k) { return total > 0 ? (double)hist[p[pl.order[k]]] / total : 0.0; };
  if (strategy == SM_STRATEGY_AUTO) {
    // Chunk-test hit rates (i.i.d. estimate from the histogram): FILTER queues the 16-byte
    // chunks holding p[pi(1)] (h1), PAIR those with a pi(1)&pi(2) survivor (h12); each
    // queued chunk costs a gather + two exact compares.  BLOCK (Alg. 4 over warp-blocks)
    // has a flat cost and wins only when even the pair test passes most chunks (m >= 3).
    // Crossovers measured on B200 (tools/pair_sweep.sh, profiles/strategy_r1.md).
    const double f1 = freq(0), f12 = m >= 2 ? f1 * freq(1) : f1;
    auto pow16 = [](double x) { x *= x; x *= x; x *= x; return x * x; };
    const double h1 = 1.0 - pow16(1.0 - f1), h12 = 1.0 - pow16(1.0 - f12);
    if (h12 > tunables().block_min_hit) {
      // m = 2: PAIR's pair test, taken per byte, is the match itself (one pass, no queue,
      // no phase B: search_impl.cuh filter_tile_q), so it replaces BLOCK at any density
      strategy = m == 2 ? kPair : kBlock;
      if (tunables().auto_packed && allow_packed) {  // small text alphabet: compare b-bit codes
        const int pk = packed();
        if (pk) strategy = pk;
      }
    } else if (m >= 2 && h1 > (m >= 32 ? tunables().pair_min_hit_long : tunables().pair_min_hit)) {
      strategy = kPair;
    } else {
      strategy = kFilter;
    }
  } else if (strategy == SM_STRATEGY_PAIR) {
    strategy = m >= 2 ? kPair : kFilter;
  } else if (strategy == SM_STRATEGY_PACKED) {
    strategy = packed();
    if (!strategy)
      return fail(SM_EINVAL, "SM_STRATEGY_PACKED needs <= 4 text symbols separable by a 1- or 2-bit field and "
                             "every pattern symbol present in the text");
    if (!allow_packed) strategy = kBlock;
  }
  pl.strategy = strategy;
  if (peel == 0) {
    // smallest r with alpha_eff * prod_{k<r} f(pi(k)) <= 1/2: the paper's reasoning
    // for r ("it is less probable that all the alpha comparisons
    // fail at the same time") at the warp's alpha_eff = 32 lanes x 16 x CPL, capped at 2048.
    double surv = std::min(32.0 * 16.0 * pl.cpl, 2048.0);
    uint32_t r = 0;
    while (r < m && surv > 0.5) surv *= freq(r++);
    const int rb = (int)r + tunables().peel_bias;  // tuning knob (0 by default)
    peel = rb < 1 ? 1u : (uint32_t)rb;
  }
  pl.r = std::min<uint32_t>(peel, (uint32_t)m);
  // FILTER: pi(1) is tested per chunk, then phase B peels pi(1) and pi(2) together
  // (filter_entry, r = 2) before the per-survivor loop
  if (pl.strategy == kFilter) pl.r = std::min<uint32_t>(2u, (uint32_t)m);
  if (pl.strategy == kPair) {
    pl.r = 2;  // pi(1), pi(2) tested together
    // PAIR's chunk test is cheaper when pi(2)'s window is word-aligned relative to
    // pi(1)'s ((a2 - a1) % 4 == 0: no funnel shifts); among the next positions whose
    // symbol is at most pair_align_slack times as frequent as pi(2)'s, move the first
    // aligned one to pi(2).  The comparison order never changes the result.
    const double slack = tunables().pair_align_slack;
    if (slack > 1.0 && !order && m >= 3) {
      const uint32_t a1 = pl.order[0];
      const double f2 = (double)hist[p[pl.order[1]]];
      for (size_t k = 1; k < m && (double)hist[p[pl.order[k]]] <= slack * f2; ++k) {
        if (((pl.order[k] - a1) & 3u) == 0) {
          std::swap(pl.order[1], pl.order[k]);
          break;
        }
      }
    }
  }
  return SM_OK;
}

sm_status host_hist(const uint8_t* t, size_t n, cudaStream_t st, uint64_t* out) {
  // the 2 KiB read-back lands in a pinned per-thread buffer (a pageable destination costs
  // a staged, synchronous copy on the step's critical path: the host plans only after it)
  static thread_local uint64_t* pinned = nullptr;
  if (!pinned) {
    void* hp = nullptr;
    if (cudaHostAlloc(&hp, 256 * sizeof(uint64_t), cudaHostAllocPortable) == cudaSuccess)
      pinned = static_cast<uint64_t*>(hp);
    else
      cudaGetLastError();  // clear it: fall back to the caller's (pageable) buffer
  }
  uint64_t* dst = pinned ? pinned : out;
  uint64_t* d = nullptr;
  SM_CUDA_TRY(pool_alloc(reinterpret_cast<void**>(&d), 256 * sizeof(uint64_t), st), "pool_alloc(hist)");
  cudaError_t e = launch_hist(t, n, d, num_sms(), st);
  if (e == cudaSuccess) {
    ++g_launches;
    e = cudaMemcpyAsync(dst, d, 256 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
  }
  cudaFreeAsync(d, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "histogram");
  if (dst != out) std::memcpy(out, dst, 256 * sizeof(uint64_t));
  return SM_OK;
}

// Descriptor of one planned pattern (see search.cuh).  `lim` = max alignments to
// count (SIZE_MAX: all n - m + 1).
void fill_desc(const Plan& pl, const uint8_t* p, size_t m, uint64_t delta, uint64_t n, uint64_t lim, uint64_t T,
               PatDesc& d, uint32_t tbl_index) {
  std::memset(&d, 0, sizeof(d));
  d.m = (uint32_t)m;
  d.r = pl.r;
  d.tbl = tbl_index;
  d.A = std::min<uint64_t>(n - m + 1, lim);
  if (pl.strategy == kFilter || pl.strategy == kPair) {  // geometry of the pi(1)-bytes
    const uint32_t a1 = pl.order[0];
    d.a1 = a1;
    d.bc1 = (uint32_t)p[a1] * 0x01010101u;
    d.pre = (a1 + 15) & ~15u;
    if (m >= 2) {
      const uint32_t a2 = pl.order[1];
      d.s2 = d.pre + a2 - a1;
      d.bc2 = (uint32_t)p[a2] * 0x01010101u;
    }
    // + 16: the pi(2) window of the last chunk reads up to 32 bytes past its base
    const uint32_t post = (((uint32_t)(m - 1 - a1) + 15) & ~15u) + 16;
    d.stage_len = (uint32_t)T + d.pre + post;
    d.k_begin = (delta + a1) / T;
    const uint64_t k_end = (delta + d.A - 1 + a1) / T + 1;
    d.ntiles = k_end - d.k_begin;
  } else {  // BLOCK and PACKED: tile in alignment space
    d.pre = 0;
    const uint32_t post = (((uint32_t)m - 1) & ~15u) + 16;
    d.stage_len = (uint32_t)T + post;
    if (is_prepacked(pl.strategy)) {
      // the stage holds code bits: (T + post') alignments x b bits, post' >= m - 1 + 64 (the
      // last unit's two-word windows), a multiple of 128 alignments (16-B granules)
      const uint32_t postp = ((uint32_t)m - 1 + 64 + 127) & ~127u;
      d.stage_len = ((uint32_t)T + postp) * (uint32_t)code_bits(pl.strategy) / 8u;
    }
    d.k_begin = 0;
    d.ntiles = (delta + d.A - 1) / T + 1;
  }
  // edge tiles: only these need range masks (tile ti covers alignments x_base + [0, T))
  const uint64_t shift = (pl.strategy == kFilter || pl.strategy == kPair) ? d.a1 : 0;
  const uint64_t first_full = (delta + shift + T - 1) / T;  // smallest k with k*T - shift >= delta
  d.edge_lo = first_full > d.k_begin ? first_full - d.k_begin : 0;
  const uint64_t kh = (delta + d.A + shift) / T;             // smallest k with (k+1)*T - shift > delta + A
  d.edge_hi = kh > d.k_begin ? kh - d.k_begin : 0;
}

struct Planned {
  Plan pl;
  const uint8_t* p;
  size_t m;
  uint64_t* count_out;
};

// kernel-parameter table entries of a planned pattern: its m (offset, symbol) pairs in pi order
size_t table_words(const Planned& q) { return q.m; }

// Build one launch over patterns `ps` (same strategy; <= kMaxBatch, table <= kTableLarge).
// The tile is the plan's (large texts: 32 KiB); the batching loops keep a launch's
// table <= kBatchTableWords; T is halved only if fewer than 2 stages fit.
void build_launch(const std::vector<const Planned*>& ps, const uint8_t* t, size_t n, uint64_t lim, int epilogue,
                  HostLaunch& L) {
  const uintptr_t tp = reinterpret_cast<uintptr_t>(t);
  std::memset(&L.a, 0, sizeof(L.a));
  L.a.base = reinterpret_cast<const uint8_t*>(tp & ~(uintptr_t)15);
  L.a.delta = tp & 15;
  L.a.n = n;
  L.strategy = ps[0]->pl.strategy;
  L.epilogue = epilogue;
  L.e.clear();
  const bool packed = is_packed(L.strategy);
  const bool pre = is_prepacked(L.strategy);
  const uint32_t cbits = (uint32_t)code_bits(L.strategy);
  L.a.code_shift = ps[0]->pl.code_shift;
  size_t words = 0;
  for (const Planned* q : ps) words += q->m;
  L.e.reserve(words);
  for (const Planned* q : ps) {
    for (size_t k = 0; k < q->m; ++k) {
      const uint32_t sym = q->p[q->pl.order[k]];
      const uint32_t v = packed ? ((sym >> L.a.code_shift) & ((1u << cbits) - 1u)) : sym;
      L.e.push_back(q->pl.order[k] | (v << 16));
    }
  }
  L.a.npat = (uint32_t)ps.size();
  L.a.tbl_words = (uint32_t)L.e.size();
  L.a.ctr = counters_ptr();
  L.a.l2_policy = tunables().l2_policy;
  L.a.wait_ns = tunables().wait_ns;
  // reporting launches reserve the per-warp position lists
  L.a.list_off = (kTblOff + 127) & ~127u;
  // reporting: kEpiStage keeps one 32 CPL-mask bitmap per warp (<= 512 B), the overflow
  // pass (kEpiWrite) a kListCap-entry position list per warp
  const uint32_t list_bytes = is_count_epi(epilogue) ? 0u
                              : epilogue == kEpiStage ? (uint32_t)(kConsumerWarps * 32 * 8 * 2)
                                                      : (uint32_t)(kConsumerWarps * kListCap * 2);
  L.a.pack_off = (L.a.list_off + list_bytes + 127) & ~127u;
  L.a.ring_off = L.a.pack_off;
  uint32_t T = ps[0]->pl.tile;
  for (;;) {
    L.a.tile = T;
    L.cpl = (int)(T / (16u * kLanesPerTilePass));
    L.d.resize(ps.size());
    uint64_t work = 0;
    uint32_t max_stage = 0, tbl = 0;
    for (size_t i = 0; i < ps.size(); ++i) {
      const Planned& q = *ps[i];
      fill_desc(q.pl, q.p, q.m, L.a.delta, n, lim, T, L.d[i], tbl);
      tbl += table_words(q);
      work += L.d[i].ntiles;
      L.d[i].work_end = work;
      L.d[i].count_out = q.count_out;
      // consecutive passes over the same text alternate direction, so each pass starts on
      // the tiles the previous one read last (still in the 126 MB L2); never changes results
      L.d[i].flags = tunables().alternate ? (uint32_t)(i & 1) : 0u;
      max_stage = std::max(max_stage, L.d[i].stage_len);
    }
    L.a.total_work = work;
    L.a.stage_stride = (max_stage + 127) & ~127u;
    if (packed && !pre) {  // double-buffered code array: 2b bytes of codes per 16-byte chunk (+ a slack word)
      L.a.pack_bytes = ((max_stage / 16u) * 2u * cbits + 16u + 127u) & ~127u;
      L.a.ring_off = L.a.pack_off + 2 * L.a.pack_bytes;
    }
    // shared memory per SM: 228 KiB, 1 KiB reserved per resident CTA
    int ctas = pre ? tunables().ctas_pre : tunables().ctas_per_sm;
    uint32_t stages = 0;
    for (; ctas >= 1; --ctas) {
      const uint32_t budget = std::min<uint32_t>(227 * 1024, 233472 / ctas - 1024);
      stages = budget > L.a.ring_off ? (budget - L.a.ring_off) / L.a.stage_stride : 0;
      if (stages >= 2) break;
    }
    if (ctas < 1) ctas = 1;
    if (stages < 2 && T > 4096) {  // only a single very long pattern can get here
      T /= 2;
      continue;
    }
    if (packed) {
      // PACKED: all r peeled steps run, so move the ones whose code window
      // is register-resident (off < 32 for 1-bit codes in 32-alignment units, else < 16)
      // to the front (stable) and tell the kernel how many: two branch-free loops
      const uint32_t lim = (cbits == 1 && L.cpl >= 2) ? 32u : 16u;
      for (size_t i = 0; i < ps.size(); ++i) {
        PatDesc& d = L.d[i];
        uint32_t* e = L.e.data() + d.tbl;
        std::stable_partition(e, e + d.r, [&](uint32_t x) { return (x & 0xFFFFu) < lim; });
        uint32_t r1 = 0;
        while (r1 < d.r && (e[r1] & 0xFFFFu) < lim) ++r1;
        d.flags |= std::min<uint32_t>(r1, 255u) << 8;
        // 1-bit codes, 32-alignment words (search_impl.cuh packed_tile, kWide): entry =
        // offset | (1 - code) << 31, so a step gets its all-0 / all-1 mask word with ONE
        // arithmetic shift (F &= window ^ mask) and uses the entry itself as the funnel-shift
        // amount (mod 32)
        if (cbits == 1 && L.cpl >= 2)
          for (uint32_t j = 0; j < d.m; ++j) e[j] = (e[j] & 0xFFFFu) | ((((e[j] >> 16) & 1u) ^ 1u) << 31);
      }
    }
    L.a.stages = std::min<uint32_t>(stages, pre ? tunables().max_stages_pre : tunables().max_stages);
    L.smem = (size_t)L.a.ring_off + (size_t)L.a.stages * L.a.stage_stride;
    const uint64_t sms = (uint64_t)num_sms();
    L.grid = (int)std::min<uint64_t>(work, sms * (uint64_t)ctas);
    if (L.grid < 1) L.grid = 1;
    return;
  }
}

sm_status launch_checked(const HostLaunch& L, cudaStream_t st, const char* what) {
  SM_CUDA_TRY(launch_search(L, st), what);
  ++g_launches;
  return SM_OK;
}

// Counts of P patterns over one text in as few launches as the batch limits allow
// (each launch runs every one of its patterns as a full pass over the text).
// order / peel: the caller's comparison order and peeling factor (P == 1 only).
// Host-side phase timing of one count call (SMGPU_HOST_TIMING=1: one line per call on
// stderr, microseconds) -- for the small-text regime where the host enqueue bounds the
// step (c1).
struct HostTiming {
  using clk = std::chrono::steady_clock;
  bool on;
  clk::time_point t0, last;
  double prep = 0, plan = 0, build = 0, launch = 0;
  int launches = 0;
  HostTiming() {
    static const bool enabled = [] {
      const char* e = std::getenv("SMGPU_HOST_TIMING");
      return e && std::atoi(e) != 0;
    }();
    on = enabled;
    if (on) t0 = last = clk::now();
  }
  double lap() {
    const auto now = clk::now();
    const double us = std::chrono::duration<double, std::micro>(now - last).count();
    last = now;
    return us;
  }
  void report(size_t P) {
    if (!on) return;
    const double tot = std::chrono::duration<double, std::micro>(clk::now() - t0).count();
    std::fprintf(stderr, "smgpu host: P=%zu total=%.1f prep=%.1f plan=%.1f build=%.1f launch=%.1f launches=%d\n", P,
                 tot, prep, plan, build, launch, launches);
  }
};

// orders / peels: the caller's comparison orders (concatenated, m[i] entries each) and
// peeling factors (0 = auto), or nullptr for the rarest-first order / auto r.
// mc / done (NEXT-4): every launch also adds its patterns' counts to mc[i] through the
// last-CTA epilogue (search_impl.cuh nvls_epilogue); done = >= 2 (P + 8) zeroed u32.
sm_status enqueue_count_batch(const uint8_t* const* ps, const size_t* ms, size_t P, const uint8_t* t, size_t n,
                              uint64_t lim, const uint64_t* hist, int strategy, uint64_t* d_counts,
                              cudaStream_t st, const uint32_t* orders = nullptr, const uint32_t* peels = nullptr,
                              uint64_t* mc = nullptr, unsigned int* done = nullptr) {
  if (P == 0) return SM_OK;
  HostTiming ht;
  SM_CUDA_TRY(cudaMemsetAsync(d_counts, 0, P * sizeof(uint64_t), st), "cudaMemsetAsync(counts)");
  uint64_t hb[256];
  const uint64_t* h = hist;
  const bool trusted = hist == nullptr;  // the histogram is computed here, from t
  if (!h) {
    sm_status s = host_hist(t, n, st, hb);
    if (s != SM_OK) return s;
    h = hb;
  }
  // NEXT-3: a <= 4-symbol text is packed once for the whole batch (on a caller histogram:
  // for any P, with the device support check and the guarded fallback, see prepack_text)
  int cb = 0;
  uint32_t* guard = nullptr;
  cudaError_t pe = cudaSuccess;
  CodeArray codes{prepack_text(h, t, n, P, !trusted, st, &cb, &guard, &pe), st};
  if (pe != cudaSuccess) return cuda_fail(pe, "prepack");
  const bool allow_packed = trusted || codes.p != nullptr;
  // plan and launch as we go: a batch is launched as soon as it is full, so the GPU
  // starts on the first patterns while the host still orders the later ones
  const TextInfo tinfo = text_info(h, n, P);
  // counter-dispatched work items for long calls: one zeroed counter per launch
  // (a call makes at most 2 (P + 7) launches: every flush holds >= 1 pattern, and a
  // guarded PACKED launch has a fallback launch)
  unsigned long long* work = nullptr;
  size_t nwork = 0, used_work = 0;
  if (use_dispatch(n, P)) {
    nwork = 2 * (P + 8);
    SM_CUDA_TRY(pool_alloc(reinterpret_cast<void**>(&work), nwork * 8, st), "pool_alloc(work counters)");
    cudaError_t e = cudaMemsetAsync(work, 0, nwork * 8, st);
    if (e != cudaSuccess) {
      cudaFreeAsync(work, st);
      return cuda_fail(e, "cudaMemsetAsync(work counters)");
    }
  }
  struct FreeWork {
    unsigned long long* p;
    cudaStream_t st;
    ~FreeWork() {
      if (p) cudaFreeAsync(p, st);
    }
  } free_work{work, st};
  size_t used_done = 0;
  if (ht.on) ht.prep += ht.lap();
  std::vector<Planned> plans(P), fallback(guard ? P : 0);
  constexpr int kStrategies = 8;                  // index = strategy value (1..7)
  std::vector<const Planned*> batch[2][kStrategies];  // [0]: plans, [1]: guarded fallbacks
  size_t words[2][kStrategies] = {};
  auto flush = [&](int fb, int strat) -> sm_status {
    if (batch[fb][strat].empty()) return SM_OK;
    if (ht.on) ht.plan += ht.lap();
    HostLaunch L;
    build_launch(batch[fb][strat], t, n, lim, mc ? kEpiCountMc : kEpiCount, L);
    L.a.codes = codes.p;
    if (guard && (fb || is_prepacked(strat))) {
      L.a.guard = guard;
      L.a.guard_mode = fb ? kGuardSet : kGuardClear;
    }
    if (work && used_work < nwork && L.a.total_work < kNoItem) L.a.work_ctr = work + used_work++;
    if (mc) {
      static const bool emulate = [] {
        const char* e = std::getenv("SMGPU_NVLS_EMULATE");
        return e && std::atoi(e) != 0;
      }();
      L.a.mc_base = mc;
      L.a.local_base = d_counts;
      L.a.done_ctr = done + used_done++;
      L.a.mc_emulate = emulate ? 1u : 0u;
    }
    batch[fb][strat].clear();
    words[fb][strat] = 0;
    if (ht.on) ht.build += ht.lap();
    const sm_status ls = launch_checked(L, st, fb ? "search kernel (guarded fallback)" : "search kernel (batch)");
    if (ht.on) {
      ht.launch += ht.lap();
      ++ht.launches;
    }
    return ls;
  };
  auto add = [&](int fb, const Planned& q) -> sm_status {
    const int k = q.pl.strategy;
    if (batch[fb][k].size() == (size_t)kMaxBatch || words[fb][k] + table_words(q) > (size_t)kBatchTableWords) {
      sm_status s = flush(fb, k);
      if (s != SM_OK) return s;
    }
    batch[fb][k].push_back(&q);
    words[fb][k] += table_words(q);
    return SM_OK;
  };
  size_t order_at = 0;
  for (size_t i = 0; i < P; ++i) {
    const uint32_t* order = orders ? orders + order_at : nullptr;
    const uint32_t peel = peels ? peels[i] : 0u;
    order_at += ms[i];
    if (n < ms[i] || lim == 0) continue;  // count stays 0
    Planned& q = plans[i];
    q = Planned{Plan(), ps[i], ms[i], d_counts + i};
    sm_status s = make_plan(ps[i], ms[i], n, h, order, peel, strategy, q.pl, &tinfo, allow_packed);
    if (s != SM_OK) return s;
    use_codes(codes, cb, q.pl);
    if (guard && is_prepacked(q.pl.strategy)) {  // its byte-compare twin, run only if the check fails
      Planned& f = fallback[i];
      f = Planned{Plan(), ps[i], ms[i], d_counts + i};
      s = make_plan(ps[i], ms[i], n, h, order, peel, strategy, f.pl, &tinfo, false);
      if (s == SM_OK) s = add(1, f);
      if (s != SM_OK) return s;
    }
    s = add(0, q);
    if (s != SM_OK) return s;
  }
  for (int fb = 0; fb < 2; ++fb)
    for (int k = 1; k < kStrategies; ++k) {
      sm_status s = flush(fb, k);
      if (s != SM_OK) return s;
    }
  ht.report(P);
  return SM_OK;
}

sm_status enqueue_count(const uint8_t* p, size_t m, const uint8_t* t, size_t n, const uint64_t* hist,
                        const uint32_t* order, uint32_t peel, int strategy, uint64_t* d_count, cudaStream_t st) {
  const uint8_t* ps[1] = {p};
  const size_t ms[1] = {m};
  return enqueue_count_batch(ps, ms, 1, t, n, UINT64_MAX, hist, strategy, d_count, st, order, &peel);
}

// Staging pool of the reporting pass (bytes).  Records: at most 16 B per reported
// position (a sparse record = 16-B header + 16-B list per match) and at most one
// 528-B bitmap record per warp-tile; plus, per launch, one partly used 8 KiB chunk
// per resident compare warp (a warp's chunk is not handed on to the next launch);
// 64 MiB slack; at most 4 GiB.  SMGPU_STAGE_BYTES overrides (tests force the overflow
// path with a tiny pool).  Tiles whose record does not fit are recomputed from the
// text by the overflow pass, so the size never changes results (the memory is
// allocated per call from the stream-ordered pool, not written beyond what is used).
uint64_t stage_pool_bytes(uint64_t cap, uint64_t items, uint64_t launches) {
  static const long long env = [] {
    const char* e = std::getenv("SMGPU_STAGE_BYTES");
    return e ? std::atoll(e) : -1LL;
  }();
  const uint64_t warps = (uint64_t)num_sms() * 4u * kConsumerWarps;  // >= resident compare warps
  // per position: <= 16 B as a list record; a bitmap record (528 B) holds > list_max of them
  const uint64_t per_pos = std::max<uint64_t>(16, (528 + tunables().list_max) / (tunables().list_max + 1ull) + 16);
  const uint64_t records = std::min<uint64_t>(per_pos * cap, items * kConsumerWarps * 528ull);
  const uint64_t partial = launches * warps * (uint64_t)kStageChunk * 16u;
  uint64_t b = env >= 0 ? (uint64_t)env : std::min<uint64_t>(4ull << 30, (64ull << 20) + records + partial);
  return (b + 15) & ~15ull;
}

// Reporting (A8) for P patterns, output concatenated in pattern order: pattern k's
// ascending positions at pos[off_k ..), off_k = sum of earlier counts (first `cap`
// positions overall are written).  One read of the text per pattern:
//   pass 1 (kEpiStage): per-(item, warp) counts + per-pattern totals, and each warp's
//          matches in an item staged as a compact record (u16 list / bitmap) in the
//          warp's own chunk of the staging pool;
//   one exclusive scan over all work items (pattern-major in caller order);
//   expand: records -> positions at the scanned offsets;
//   overflow pass (kEpiWrite): tiles whose record did not fit the pool, recomputed
//          from the text (no work at all when the pool sufficed).
// cap == 0 (the two-call idiom's first call): counts only.
sm_status enqueue_report_batch(const uint8_t* const* ps, const size_t* ms, size_t P, const uint8_t* t, size_t n,
                               uint64_t lim, const uint64_t* hist, const uint32_t* order, uint32_t peel,
                               int strategy, uint64_t* pos, size_t cap, uint64_t* d_counts, uint64_t pos_offset,
                               cudaStream_t st) {
  if (P == 0) return SM_OK;
  SM_CUDA_TRY(cudaMemsetAsync(d_counts, 0, P * sizeof(uint64_t), st), "cudaMemsetAsync(counts)");
  uint64_t hb[256];
  const uint64_t* h = hist;
  uint32_t sh_unused = 0;
  // PACKED is exact only on a code field injective on t's own symbols: when a caller
  // histogram (frequencies may come from another corpus) would select it,
  // reporting takes its strategy and order from t's device histogram instead
  const bool may_pack = strategy == SM_STRATEGY_PACKED || (strategy == SM_STRATEGY_AUTO && tunables().auto_packed);
  if (!h || (may_pack && text_code_bits(h, &sh_unused) != 0)) {
    sm_status s = host_hist(t, n, st, hb);
    if (s != SM_OK) return s;
    h = hb;
  }
  int cb = 0;
  uint32_t* no_guard = nullptr;
  cudaError_t pe = cudaSuccess;
  CodeArray codes{prepack_text(h, t, n, P, false, st, &cb, &no_guard, &pe), st};
  if (pe != cudaSuccess) return cuda_fail(pe, "prepack");
  const TextInfo tinfo = text_info(h, n, P);
  const int epi1 = cap > 0 ? kEpiStage : kEpiCount;
  // Patterns are planned in caller order and launched in strategy batches as soon as a
  // batch is full, so the GPU starts while the host still orders later patterns.  Each
  // pattern's work items get the slots [item_base, item_base + ntiles) of the per-item
  // arrays, item_base = the prefix of the EARLIER patterns' tile counts (known when its
  // batch launches), so one scan still yields the concatenated, pattern-ordered layout.
  // The scratch is sized before the first launch with each pattern's largest possible
  // tile count at the planned tile size.
  const uint64_t T0 = tinfo.tiling.tile;
  const uintptr_t tp = reinterpret_cast<uintptr_t>(t);
  const uint64_t nt_max = ((tp & 15) + n + T0 - 1) / T0 + 2;
  uint64_t items_max = 0;
  for (size_t i = 0; i < P; ++i)
    if (!(n < ms[i] || lim == 0)) items_max += nt_max;
  if (items_max == 0) return SM_OK;
  if (items_max >= (1ull << 31)) return fail(SM_EINVAL, "report: 2^31 or more (pattern, tile) work items in one call");
  const uint64_t nL_max = (P + kMaxBatch - 1) / kMaxBatch + 16;  // typical launch count (+ slack)
  size_t temp_bytes = 0;
  SM_CUDA_TRY(exclusive_scan_wc(nullptr, nullptr, items_max, nullptr, &temp_bytes, st), "scan sizing");
  auto al = [](uint64_t b) { return (b + 255) & ~255ull; };
  uint8_t* scratch = nullptr;
  uint16_t* wc = nullptr;
  uint32_t *ovf_bits = nullptr, *ovf_n = nullptr, *ovf_items = nullptr;
  unsigned long long *stage_used = nullptr, *expand_work = nullptr, *work = nullptr;
  uint64_t* offsets = nullptr;
  void* temp = nullptr;
  uint8_t* stage = nullptr;
  uint64_t stage_cap16 = 0;
  const size_t max_launches = 2 * P + 16;  // every flush holds >= 1 pattern
  cudaError_t e = cudaSuccess;
  if (cap > 0) {
    const uint64_t wc_b = al(items_max * 16), offs_b = al(items_max * 8), bits_b = al((items_max + 31) / 32 * 4),
                   ovf_b = al(items_max * 4), ctr_b = al(16 + max_launches * 12), temp_b = al(temp_bytes),
                   stage_b = stage_pool_bytes(cap, items_max, nL_max);
    SM_CUDA_TRY(pool_alloc(reinterpret_cast<void**>(&scratch),
                           wc_b + bits_b + ctr_b + offs_b + ovf_b + temp_b + stage_b, st),
                "pool_alloc(report scratch)");
    uint8_t* q = scratch;  // zero-initialised part first: wc, ovf_bits, counters
    wc = reinterpret_cast<uint16_t*>(q); q += wc_b;
    ovf_bits = reinterpret_cast<uint32_t*>(q); q += bits_b;
    stage_used = reinterpret_cast<unsigned long long*>(q);
    expand_work = stage_used + 1;
    work = reinterpret_cast<unsigned long long*>(q + 16);  // [max_launches] pass-1 dispatch counters
    ovf_n = reinterpret_cast<uint32_t*>(q + 16 + max_launches * 8); q += ctr_b;
    offsets = reinterpret_cast<uint64_t*>(q); q += offs_b;
    ovf_items = reinterpret_cast<uint32_t*>(q); q += ovf_b;
    temp = q; q += temp_b;
    stage = q;
    // whole chunks only: every chunk a warp claims can hold the largest record plus its
    // terminator, so no claimed chunk is ever left without a terminator header
    stage_cap16 = stage_b / 16 / kStageChunk * kStageChunk;
    e = cudaMemsetAsync(scratch, 0, wc_b + bits_b + ctr_b, st);
    if (e != cudaSuccess) {
      cudaFreeAsync(scratch, st);
      return cuda_fail(e, "cudaMemsetAsync(report scratch)");
    }
  }
  struct FreeScratch {
    uint8_t* p;
    cudaStream_t st;
    ~FreeScratch() {
      if (p) cudaFreeAsync(p, st);
    }
  } free_scratch{scratch, st};
  const bool dispatch = use_dispatch(n, P);
  std::vector<Planned> plans(P);
  std::vector<std::vector<const Planned*>> runs;  // each launch's patterns (the overflow pass rebuilds)
  std::vector<std::vector<uint64_t>> run_bases;   // and their item bases
  std::vector<uint64_t> run_ovf;                  // and the offset of their overflow queue
  std::vector<const Planned*> batch[8];
  size_t words[8] = {};
  uint64_t items = 0, ovf_at = 0;
  std::vector<uint64_t> base_of(P, 0);
  auto flush = [&](int strat) -> sm_status {
    if (batch[strat].empty()) return SM_OK;
    HostLaunch L;
    build_launch(batch[strat], t, n, lim, epi1, L);
    L.a.codes = codes.p;
    std::vector<uint64_t> bases(L.d.size());
    for (size_t k = 0; k < L.d.size(); ++k) {
      const size_t i = (size_t)(L.d[k].count_out - d_counts);
      if (L.d[k].ntiles > nt_max) return fail(SM_ENOMEM, "report: tile count bound exceeded");
      L.d[k].item_base = base_of[i];
      bases[k] = base_of[i];
    }
    run_ovf.push_back(ovf_at);
    const size_t li = runs.size();
    if (cap > 0) {
      if (li >= max_launches) return fail(SM_ENOMEM, "report: launch count bound exceeded");
      L.a.wc = wc;
      L.a.stage = stage;
      L.a.stage_used = stage_used;
      L.a.stage_cap16 = stage_cap16;
      L.a.ovf_bits = ovf_bits;
      L.a.ovf_items = ovf_items + ovf_at;  // this launch's overflow queue (capacity: its items)
      L.a.ovf_n = ovf_n + li;
      L.a.pos_offset = pos_offset;
      L.a.list_max = tunables().list_max;
      if (dispatch && L.a.total_work < kNoItem) L.a.work_ctr = work + li;
      ovf_at += L.a.total_work;
    }
    runs.push_back(batch[strat]);
    run_bases.push_back(std::move(bases));
    batch[strat].clear();
    words[strat] = 0;
    return launch_checked(L, st, cap > 0 ? "search kernel (report pass 1)" : "search kernel (report totals)");
  };
  for (size_t i = 0; i < P; ++i) {
    if (n < ms[i] || lim == 0) continue;  // no alignments: count 0, no positions
    Planned& q = plans[i];
    q = Planned{Plan(), ps[i], ms[i], d_counts + i};
    sm_status s = make_plan(ps[i], ms[i], n, h, P == 1 ? order : nullptr, P == 1 ? peel : 0, strategy, q.pl,
                            &tinfo);
    if (s != SM_OK) return s;
    use_codes(codes, cb, q.pl);
    PatDesc d;  // this pattern's tile count at the launch tile size (fill_desc is what build_launch uses)
    fill_desc(q.pl, q.p, q.m, tp & 15, n, lim, T0, d, 0);
    if (d.ntiles > nt_max) return fail(SM_ENOMEM, "report: tile count bound exceeded");
    base_of[i] = items;
    items += nt_max;  // slots [base, base + ntiles) used; the rest of the pattern's slots stay zero
    const int k = q.pl.strategy;
    if (batch[k].size() == (size_t)kMaxBatch || words[k] + table_words(q) > (size_t)kBatchTableWords) {
      s = flush(k);
      if (s != SM_OK) return s;
    }
    batch[k].push_back(&q);
    words[k] += table_words(q);
  }
  for (int k = 1; k < 8; ++k) {
    sm_status s = flush(k);
    if (s != SM_OK) return s;
  }
  if (cap == 0 || runs.empty()) return SM_OK;
  e = exclusive_scan_wc(wc, offsets, items, temp, &temp_bytes, st);
  if (e == cudaSuccess) g_launches += 1;
  if (e == cudaSuccess) {
    e = launch_stage_expand(stage, stage_used, stage_cap16, wc, offsets, pos, cap, expand_work, num_sms(), st);
    if (e == cudaSuccess) ++g_launches;
  }
  for (size_t li = 0; li < runs.size(); ++li) {  // overflow pass (CTAs exit at once when the queue is empty)
    if (e != cudaSuccess) break;
    HostLaunch W;  // its own shared-memory layout (position lists), same patterns and arguments
    build_launch(runs[li], t, n, lim, kEpiWrite, W);
    for (size_t i = 0; i < W.d.size(); ++i) W.d[i].item_base = run_bases[li][i];
    W.a.codes = codes.p;
    W.a.ovf_items = ovf_items + run_ovf[li];
    W.a.ovf_n = ovf_n + li;
    W.a.pos_offset = pos_offset;
    W.a.tile_offsets = offsets;
    W.a.pos = pos;
    W.a.cap = cap;
    e = launch_search(W, st);
    if (e == cudaSuccess) ++g_launches;
  }
  if (e != cudaSuccess) return cuda_fail(e, "report");
  return SM_OK;
}

sm_status enqueue_report(const uint8_t* p, size_t m, const uint8_t* t, size_t n, const uint64_t* hist,
                         const uint32_t* order, uint32_t peel, int strategy, uint64_t* pos, size_t cap,
                         uint64_t* d_count, cudaStream_t st) {
  const uint8_t* ps[1] = {p};
  const size_t ms[1] = {m};
  return enqueue_report_batch(ps, ms, 1, t, n, UINT64_MAX, hist, order, peel, strategy, pos, cap, d_count, 0, st);
}

}  // namespace

extern "C" {

uint64_t sm_count(const uint8_t* p, size_t m, const uint8_t* t, size_t n) {
  if (check_pattern_text(p, m, t, n) != SM_OK) return SM_COUNT_ERROR;
  if (n < m) return 0;
  cudaStream_t st = cudaStreamPerThread;
  uint64_t* d = nullptr;
  cudaError_t e = pool_alloc(reinterpret_cast<void**>(&d), sizeof(uint64_t), st);
  if (e != cudaSuccess) {
    cuda_fail(e, "pool_alloc(count)");
    return SM_COUNT_ERROR;
  }
  sm_status s = enqueue_count(p, m, t, n, nullptr, nullptr, 0, SM_STRATEGY_AUTO, d, st);
  uint64_t h = SM_COUNT_ERROR;
  if (s == SM_OK) {
    e = cudaMemcpyAsync(&h, d, sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      cuda_fail(e, "sm_count");
      h = SM_COUNT_ERROR;
    }
  }
  cudaFreeAsync(d, st);
  cudaStreamSynchronize(st);
  return s == SM_OK ? h : SM_COUNT_ERROR;
}

sm_status sm_report(const uint8_t* p, size_t m, const uint8_t* t, size_t n, uint64_t* pos, size_t cap,
                    uint64_t* count_out) {
  sm_status s = check_pattern_text(p, m, t, n);
  if (s != SM_OK) return s;
  if (!count_out) return fail(SM_EINVAL, "count_out is NULL");
  if (cap > 0) {
    if (!pos) return fail(SM_EINVAL, "pos is NULL with cap > 0");
    s = check_device_ptr(pos, "pos");
    if (s != SM_OK) return s;
  }
  *count_out = 0;
  if (n < m) return SM_OK;
  cudaStream_t st = cudaStreamPerThread;
  uint64_t* d = nullptr;
  SM_CUDA_TRY(pool_alloc(reinterpret_cast<void**>(&d), sizeof(uint64_t), st), "pool_alloc(count)");
  s = enqueue_report(p, m, t, n, nullptr, nullptr, 0, SM_STRATEGY_AUTO, pos, cap, d, st);
  uint64_t h = 0;
  cudaError_t e = cudaSuccess;
  if (s == SM_OK) {
    e = cudaMemcpyAsync(&h, d, sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  cudaFreeAsync(d, st);
  cudaStreamSynchronize(st);
  if (s != SM_OK) return s;
  if (e != cudaSuccess) return cuda_fail(e, "sm_report");
  *count_out = h;
  if (h > cap) return fail(SM_ETRUNC, "more occurrences than cap; first cap positions written");
  return SM_OK;
}

sm_status sm_symbol_order(const uint8_t* t, size_t n, const uint8_t* p, size_t m, uint32_t* order) {
  sm_status s = check_pattern_text(p, m, t, n);
  if (s != SM_OK) return s;
  if (!order) return fail(SM_EINVAL, "order is NULL");
  uint64_t hb[256];
  if (n > 0) {
    s = host_hist(t, n, cudaStreamPerThread, hb);
    if (s != SM_OK) return s;
  } else {
    std::memset(hb, 0, sizeof(hb));
  }
  order_from_hist(hb, p, m, order);
  return SM_OK;
}

sm_status sm_histogram(const uint8_t* t, size_t n, uint64_t* d_hist, void* stream) {
  if (!d_hist) return fail(SM_EINVAL, "d_hist is NULL");
  sm_status s = check_device_ptr(d_hist, "d_hist");
  if (s != SM_OK) return s;
  if (n > 0) {
    if (!t) return fail(SM_EINVAL, "t is NULL with n > 0");
    s = check_device_ptr(t, "t");
    if (s != SM_OK) return s;
  }
  SM_CUDA_TRY(launch_hist(t, n, d_hist, num_sms(), as_stream(stream)), "histogram kernel");
  if (n > 0) ++g_launches;
  return SM_OK;
}

sm_status sm_order_from_histogram(const uint64_t* hist, const uint8_t* p, size_t m, uint32_t* order) {
  if (m == 0) return fail(SM_EINVAL, "m == 0");
  if (!hist || !p || !order) return fail(SM_EINVAL, "NULL argument");
  order_from_hist(hist, p, m, order);
  return SM_OK;
}

sm_status sm_count_async(const uint8_t* p, size_t m, const uint8_t* t, size_t n, const uint64_t* hist,
                         const uint32_t* order, uint32_t peel, int strategy, uint64_t* d_count, void* stream) {
  sm_status s = check_pattern_text(p, m, t, n);
  if (s != SM_OK) return s;
  if (!d_count) return fail(SM_EINVAL, "d_count is NULL");
  s = check_device_ptr(d_count, "d_count");
  if (s != SM_OK) return s;
  return enqueue_count(p, m, t, n, hist, order, peel, strategy, d_count, as_stream(stream));
}

sm_status sm_count_batch(const uint8_t* const* p, const size_t* m, size_t P, const uint8_t* t, size_t n,
                         size_t max_alignments, const uint64_t* hist, int strategy, uint64_t* d_counts,
                         void* stream) {
  if (P == 0) return SM_OK;
  if (!p || !m || !d_counts) return fail(SM_EINVAL, "NULL argument");
  if (strategy < SM_STRATEGY_AUTO || strategy > SM_STRATEGY_PAIR) return fail(SM_EINVAL, "bad strategy");
  for (size_t i = 0; i < P; ++i) {
    if (m[i] == 0) return fail(SM_EINVAL, "m[i] == 0: empty pattern is undefined (reading R2)");
    if (m[i] > SM_MAX_PATTERN) return fail(SM_EINVAL, "m[i] > SM_MAX_PATTERN (4096)");
    if (!p[i]) return fail(SM_EINVAL, "p[i] is NULL");
  }
  if (n > 0) {
    if (!t) return fail(SM_EINVAL, "t is NULL with n > 0");
    sm_status s = check_device_ptr(t, "t");
    if (s != SM_OK) return s;
  }
  sm_status s = check_device_ptr(d_counts, "d_counts");
  if (s != SM_OK) return s;
  return enqueue_count_batch(p, m, P, t, n, (uint64_t)max_alignments, hist, strategy, d_counts, as_stream(stream));
}

sm_status sm_count_batch_ordered(const uint8_t* const* p, const size_t* m, size_t P, const uint8_t* t, size_t n,
                                 size_t max_alignments, const uint64_t* hist, const uint32_t* orders,
                                 const uint32_t* peels, int strategy, uint64_t* d_counts, void* stream) {
  if (P == 0) return SM_OK;
  if (!p || !m || !d_counts) return fail(SM_EINVAL, "NULL argument");
  if (strategy < SM_STRATEGY_AUTO || strategy > SM_STRATEGY_PAIR) return fail(SM_EINVAL, "bad strategy");
  size_t at = 0;
  for (size_t i = 0; i < P; ++i) {
    if (m[i] == 0) return fail(SM_EINVAL, "m[i] == 0: empty pattern is undefined (reading R2)");
    if (m[i] > SM_MAX_PATTERN) return fail(SM_EINVAL, "m[i] > SM_MAX_PATTERN (4096)");
    if (!p[i]) return fail(SM_EINVAL, "p[i] is NULL");
    if (orders && !valid_permutation(orders + at, m[i])) return fail(SM_EINVAL, "orders[i] is not a permutation");
    at += m[i];
  }
  if (n > 0) {
    if (!t) return fail(SM_EINVAL, "t is NULL with n > 0");
    sm_status s = check_device_ptr(t, "t");
    if (s != SM_OK) return s;
  }
  sm_status s = check_device_ptr(d_counts, "d_counts");
  if (s != SM_OK) return s;
  return enqueue_count_batch(p, m, P, t, n, (uint64_t)max_alignments, hist, strategy, d_counts, as_stream(stream),
                             orders, peels);
}

sm_status sm_count_batch_multicast(const uint8_t* const* p, const size_t* m, size_t P, const uint8_t* t, size_t n,
                                   size_t max_alignments, const uint64_t* hist, int strategy, uint64_t* mc_counts,
                                   void* stream) {
  if (P == 0) return SM_OK;
  if (!p || !m || !mc_counts) return fail(SM_EINVAL, "NULL argument");
  if (strategy < SM_STRATEGY_AUTO || strategy > SM_STRATEGY_PAIR) return fail(SM_EINVAL, "bad strategy");
  for (size_t i = 0; i < P; ++i) {
    if (m[i] == 0) return fail(SM_EINVAL, "m[i] == 0: empty pattern is undefined (reading R2)");
    if (m[i] > SM_MAX_PATTERN) return fail(SM_EINVAL, "m[i] > SM_MAX_PATTERN (4096)");
    if (!p[i]) return fail(SM_EINVAL, "p[i] is NULL");
  }
  if (n > 0) {
    if (!t) return fail(SM_EINVAL, "t is NULL with n > 0");
    sm_status s = check_device_ptr(t, "t");
    if (s != SM_OK) return s;
  }
  if (reinterpret_cast<uintptr_t>(mc_counts) & 7u) return fail(SM_EINVAL, "mc_counts must be 8-byte aligned");
  cudaStream_t st = as_stream(stream);
  // this rank's counts (scratch) + one zeroed done-counter per launch (a call makes at
  // most 2 (P + 8) launches); the last CTA of each launch adds its patterns' counts to
  // mc_counts with multimem.red (search_impl.cuh nvls_epilogue)
  const size_t nd = 2 * (P + 8);
  uint8_t* scratch = nullptr;
  SM_CUDA_TRY(pool_alloc(reinterpret_cast<void**>(&scratch), P * sizeof(uint64_t) + nd * 4, st),
              "pool_alloc(counts)");
  uint64_t* local = reinterpret_cast<uint64_t*>(scratch);
  unsigned int* done = reinterpret_cast<unsigned int*>(scratch + P * sizeof(uint64_t));
  sm_status s = SM_OK;
  cudaError_t e = cudaMemsetAsync(done, 0, nd * 4, st);
  if (e != cudaSuccess) s = cuda_fail(e, "cudaMemsetAsync(done counters)");
  if (s == SM_OK)
    s = enqueue_count_batch(p, m, P, t, n, (uint64_t)max_alignments, hist, strategy, local, st, nullptr, 0,
                            mc_counts, done);
  cudaFreeAsync(scratch, st);
  return s;
}

sm_status sm_report_batch(const uint8_t* const* p, const size_t* m, size_t P, const uint8_t* t, size_t n,
                          size_t max_alignments, const uint64_t* hist, int strategy, uint64_t* pos, size_t cap,
                          uint64_t* d_counts, uint64_t position_offset, void* stream) {
  if (P == 0) return SM_OK;
  if (!p || !m || !d_counts) return fail(SM_EINVAL, "NULL argument");
  if (strategy < SM_STRATEGY_AUTO || strategy > SM_STRATEGY_PAIR) return fail(SM_EINVAL, "bad strategy");
  for (size_t i = 0; i < P; ++i) {
    if (m[i] == 0) return fail(SM_EINVAL, "m[i] == 0: empty pattern is undefined (reading R2)");
    if (m[i] > SM_MAX_PATTERN) return fail(SM_EINVAL, "m[i] > SM_MAX_PATTERN (4096)");
    if (!p[i]) return fail(SM_EINVAL, "p[i] is NULL");
  }
  if (n > 0) {
    if (!t) return fail(SM_EINVAL, "t is NULL with n > 0");
    sm_status s = check_device_ptr(t, "t");
    if (s != SM_OK) return s;
  }
  sm_status s = check_device_ptr(d_counts, "d_counts");
  if (s != SM_OK) return s;
  if (cap > 0) {
    if (!pos) return fail(SM_EINVAL, "pos is NULL with cap > 0");
    s = check_device_ptr(pos, "pos");
    if (s != SM_OK) return s;
  }
  return enqueue_report_batch(p, m, P, t, n, (uint64_t)max_alignments, hist, nullptr, 0, strategy, pos, cap,
                              d_counts, position_offset, as_stream(stream));
}

sm_status sm_report_async(const uint8_t* p, size_t m, const uint8_t* t, size_t n, const uint64_t* hist,
                          const uint32_t* order, uint32_t peel, int strategy, uint64_t* pos, size_t cap,
                          uint64_t* d_count, void* stream) {
  sm_status s = check_pattern_text(p, m, t, n);
  if (s != SM_OK) return s;
  if (!d_count) return fail(SM_EINVAL, "d_count is NULL");
  s = check_device_ptr(d_count, "d_count");
  if (s != SM_OK) return s;
  if (cap > 0) {
    if (!pos) return fail(SM_EINVAL, "pos is NULL with cap > 0");
    s = check_device_ptr(pos, "pos");
    if (s != SM_OK) return s;
  }
  return enqueue_report(p, m, t, n, hist, order, peel, strategy, pos, cap, d_count, as_stream(stream));
}

sm_status sm_heuristic_order(const uint8_t* p, size_t m, int kind, uint8_t space, uint32_t* order) {
  if (m == 0 || !order || (kind != SM_ORDER_IDENTITY && !p)) return fail(SM_EINVAL, "bad arguments to sm_heuristic_order");
  if (kind == SM_ORDER_IDENTITY) {
    for (size_t j = 0; j < m; ++j) order[j] = (uint32_t)j;
    return SM_OK;
  }
  if (kind != SM_ORDER_PI_H && kind != SM_ORDER_PI_HS) return fail(SM_EINVAL, "unknown order kind");
  // positions taking part in the pi_h traversal: all (pi_h) or the non-space ones (pi_hs)
  std::vector<uint32_t> R;
  for (size_t j = 0; j < m; ++j)
    if (kind == SM_ORDER_PI_H || p[j] != space) R.push_back((uint32_t)j);
  // pi_h over R by rank: first, last, then stride-3 chains from the
  // 4th, 3rd, 2nd element (1-based), skipping ranks already taken (reading R18)
  const size_t r = R.size();
  std::vector<char> used(r + 1, 0);
  size_t k = 0;
  auto take = [&](size_t rank1) {  // 1-based rank
    if (rank1 >= 1 && rank1 <= r && !used[rank1]) {
      used[rank1] = 1;
      order[k++] = R[rank1 - 1];
    }
  };
  if (r) {
    take(1);
    take(r);
    for (size_t start : {4, 3, 2})
      for (size_t q = start; q <= r; q += 3) take(q);
  }
  if (kind == SM_ORDER_PI_HS)  // spaces last, ascending
    for (size_t j = 0; j < m; ++j)
      if (p[j] == space) order[k++] = (uint32_t)j;
  return SM_OK;
}

sm_status sm_plan(const uint8_t* p, size_t m, const uint64_t* hist, const uint32_t* order, uint32_t peel,
                  int strategy, int* strategy_out, uint32_t* peel_out) {
  if (m == 0 || m > SM_MAX_PATTERN || !p || !hist) return fail(SM_EINVAL, "bad arguments to sm_plan");
  uint64_t n = 0;
  for (int c = 0; c < 256; ++c) n += hist[c];
  Plan pl;
  sm_status s = make_plan(p, m, n, hist, order, peel, strategy, pl);
  if (s != SM_OK) return s;
  if (strategy_out) *strategy_out = pl.strategy;
  if (peel_out) *peel_out = pl.r;
  return SM_OK;
}

sm_status sm_last_error(void) { return g_status; }
const char* sm_last_error_message(void) { return g_message.c_str(); }
void sm_clear_error(void) {
  g_status = SM_OK;
  g_message.clear();
}

const char* sm_status_string(sm_status s) {
  switch (s) {
    case SM_OK: return "SM_OK";
    case SM_EINVAL: return "SM_EINVAL";
    case SM_ETRUNC: return "SM_ETRUNC";
    case SM_ENOMEM: return "SM_ENOMEM";
    case SM_ECUDA: return "SM_ECUDA";
  }
  return "SM_UNKNOWN";
}

sm_status sm_counters(uint64_t* out, int reset) {
  if (!out) return fail(SM_EINVAL, "out is NULL");
  unsigned long long* d = counters_ptr();
  if (!d) return fail(SM_EINVAL, "not the instrumented build (libsmgpu_counters.so, -DSMGPU_COUNTERS)");
  SM_CUDA_TRY(cudaDeviceSynchronize(), "sm_counters sync");
  SM_CUDA_TRY(cudaMemcpy(out, d, kCounters * sizeof(uint64_t), cudaMemcpyDeviceToHost), "sm_counters copy");
  if (reset) SM_CUDA_TRY(cudaMemset(d, 0, kCounters * sizeof(uint64_t)), "sm_counters reset");
  return SM_OK;
}

sm_status sm_trim_scratch(size_t keep_bytes) {
  int dev = 0;
  SM_CUDA_TRY(cudaGetDevice(&dev), "cudaGetDevice");
  cudaMemPool_t pool = nullptr;
  {
    std::lock_guard<std::mutex> g(g_pool_mu);
    if (dev >= 0 && dev < 64) pool = g_pools[dev];
  }
  if (!pool) return SM_OK;  // nothing allocated on this device yet
  SM_CUDA_TRY(cudaDeviceSynchronize(), "sm_trim_scratch sync");
  SM_CUDA_TRY(cudaMemPoolTrimTo(pool, keep_bytes), "cudaMemPoolTrimTo");
  return SM_OK;
}

const char* sm_version(void) {
#ifdef SMGPU_COUNTERS
  return "smgpu 0.1 (sm_100a, compare counters)";
#else
  return "smgpu 0.1 (sm_100a)";
#endif
}
uint64_t sm_launch_count(void) { return g_launches; }

}  // extern "C"
