// runtime.cu -- host runtime and C ABI of libsieve.so (include/sieve.h).
//
// Responsibilities: argument validation (error codes of sieve.h), planning of
// a call (step A1: odd-only grid, segments, grid size), device scratch owned
// by the library, stream handling, host<->device staging for host outputs,
// and the launch sequences of the three north_star calls.  Each is ONE sieve
// launch: the base primes (A2) are computed inside it (fused A2, a
// cooperative launch with two grid barriers), then
//   count  : A3-A6, the last CTA reduces the per-CTA (count, sum)
//   bitmap : A3-A7, the fused write-back: in-register transpose, count,
//            one TMA bulk copy per warp's 16 blocks to HBM
//   primes : A3, A4/A5, A8 per-segment decoupled look-back + compaction
// When the cooperative launch is not possible (a slice of the odd numbers
// <= r does not fit a segment, or the launch is refused) the base-prime
// kernel K1 runs first and the sieve is an ordinary launch.
// No C++ exception crosses the ABI; there is no CPU fallback.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sieve.h"
#include "internal.h"
#include "peer.cuh"

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
std::atomic<uint64_t> g_coop_fallbacks{0};  // refused cooperative launches (diagnostics)

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CUDA_TRY(expr)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? SIEVE_ENOMEM : SIEVE_ECUDA,          \
                  "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define TRY(expr)           \
  do {                      \
    int rc_ = (expr);       \
    if (rc_ < 0) return rc_; \
  } while (0)

// exact integer square root (largest r with r*r <= x), x < 2^64
uint64_t isqrt_u64(uint64_t x) {
  uint64_t r = (uint64_t)std::sqrt((double)x);
  while (r > 0 && r * r > x) --r;
  while ((r + 1) * (r + 1) <= x) ++r;
  return r;
}

struct Plan {           // step A1 for one range [lo, hi)
  uint64_t lo = 0, hi = 0;
  uint64_t o0 = 1;      // lo | 1
  uint64_t nbits = 0;   // odd slots B
  uint64_t words = 0;   // ceil(B/32)
  uint64_t nseg = 0;    // ceil(B/S)
  uint64_t r = 0;       // isqrt(hi-1)
  bool two = false;     // 2 in [lo, hi)
  uint64_t sbits = 0;   // segment size S (odd slots) of this call
};

template <typename T>
struct DevBuf {
  T *p = nullptr;
  size_t n = 0;
  int ensure(size_t need) {
    if (need <= n) return 0;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    size_t want = std::max(need, n + n / 2);
    cudaError_t e = cudaMalloc(&p, want * sizeof(T));
    if (e != cudaSuccess) {
      e = cudaMalloc(&p, need * sizeof(T));
      if (e != cudaSuccess) {
        p = nullptr;
        return fail(SIEVE_ENOMEM, "cudaMalloc(%zu bytes) failed: %s", need * sizeof(T),
                    cudaGetErrorString(e));
      }
      want = need;
    }
    n = want;
    return 0;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

struct Ctx {
  std::mutex mu;
  int device = -1;
  bool ready = false;
  int nsm = 0;
  cudaStream_t own = nullptr;
  cudaStream_t user = nullptr;
  bool user_set = false;
  sieve_options opt{};
  size_t smem_limit_set = 0;
  size_t occ_key = 0;  // (shared memory, threads) of the cached occupancy
  int occ = 0;
  DevBuf<uint32_t> tables;
  DevBuf<uint32_t> primes;
  DevBuf<uint64_t> recips;
  DevBuf<uint2> pk44;  // batch: {p, floor(2^44/p)} of the library-owned base primes
  DevBuf<uint32_t> nbase;
  DevBuf<uint64_t> partials;
  DevBuf<unsigned int> done;
  DevBuf<uint64_t> result;
  DevBuf<uint32_t> bitmap;
  DevBuf<uint64_t> list;
  DevBuf<sv::BatchItem> items;
  DevBuf<uint64_t> bres;
  DevBuf<uint64_t> blo, bhi;        // batch: the intervals, on the device
  DevBuf<uint32_t> plan;            // batch: class histogram + cursors (hist kept zero)
  DevBuf<uint32_t> nitems;          // batch: the planned item count
  DevBuf<uint2> buckets;  // step A5 bucket rings
  DevBuf<uint64_t> kflags;  // K1 look-back flags (epoch-tagged, never reset)
  uint32_t epoch = 0;
  DevBuf<uint32_t> bcounts;    // fused A2: per-CTA prime counts
  DevBuf<unsigned int> gbar;   // fused A2: grid barrier counter (kept 0 between launches)
  DevBuf<unsigned long long> lflags;  // list-mode look-back flags (epoch-tagged)
  uint32_t lepoch = 0;
  uint64_t *h_res = nullptr;  // pinned [2]
  unsigned long long *prof = nullptr;  // diagnostics: phase-cycle counters
  uint32_t flags = 0;                  // diagnostics: sv::kFlagSkipMarking
  // F4 fused all-reduce (peer.cuh): this process's slab, the peers' slabs
  // opened from their IPC handles, and the device array of all ranks' slabs
  struct Peers {
    unsigned long long *slab = nullptr;  // own slab (library-allocated, IPC-exported)
    std::vector<void *> opened;          // peer slabs opened by sieve_peer_attach
    DevBuf<unsigned long long *> ptrs;   // [world]
    uint32_t world = 0, rank = 0;        // world == 0: not attached
    uint64_t epoch = 0;                  // fused launches since the attach
    uint64_t timeout_ns = 0;
  } peer;
  cudaStream_t stream() const { return user_set ? user : own; }
};

Ctx g;
constexpr size_t kMaxDynSmem = 227 * 1024 - 1024;  // per-block limit minus static shared memory

void default_options(sieve_options &o) {
  memset(&o, 0, sizeof o);
  o.segment_kb = SIEVE_DEFAULT_SEGMENT_KB;
  o.wheel = SIEVE_DEFAULT_WHEEL;  // A/B with the skip of multiples of 3 and 5: 31 beats 41 by 1.4-1.8 %
  o.ctas_per_sm = 0;
  o.threads = SIEVE_MAX_THREADS;
}

int ng_for_wheel(uint32_t w) {
  switch (w) {
    case 11: return 1;
    case 17: return 2;
    case 23: return 3;
    case 31: return 4;
    case 41: return 5;
    case 47: return 6;
    default: return -1;
  }
}

// transposed word table g (internal.h): TT[y] bit i = 1 iff 2x+1 is divisible
// by a prime of group g, x = (y + 32 i) mod P_g
void build_tables(std::vector<uint32_t> &t) {
  static const uint32_t groups[sv::kMaxGroups][4] = {
      {3, 5, 7, 11}, {13, 17, 0, 0}, {19, 23, 0, 0}, {29, 31, 0, 0}, {37, 41, 0, 0}, {43, 47, 0, 0}};
  t.assign(sv::tables_words(sv::kMaxGroups), 0u);
  for (int g = 0; g < sv::kMaxGroups; ++g) {
    const uint32_t P = sv::group_period(g);
    uint32_t *w = t.data() + sv::group_offset(g);
    for (uint32_t y = 0; y < P; ++y)
      for (uint32_t i = 0; i < 32; ++i) {
        const uint64_t x = (y + 32ull * i) % P;
        const uint64_t n = 2 * x + 1;
        bool hit = false;
        for (int q = 0; q < 4 && groups[g][q]; ++q) hit |= (n % groups[g][q]) == 0;
        if (hit) w[y] |= 1u << i;
      }
  }
}

int ensure_ready() {
  if (g.ready) return 0;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev <= 0)
    return fail(SIEVE_ENODEV, "no CUDA device available (%s)", cudaGetErrorString(e));
  if (g.device < 0) CUDA_TRY(cudaGetDevice(&g.device));
  CUDA_TRY(cudaSetDevice(g.device));
  CUDA_TRY(cudaDeviceGetAttribute(&g.nsm, cudaDevAttrMultiProcessorCount, g.device));
  if (!g.own) CUDA_TRY(cudaStreamCreateWithFlags(&g.own, cudaStreamNonBlocking));
  if (g.opt.segment_kb == 0) default_options(g.opt);
  std::vector<uint32_t> t;
  build_tables(t);
  TRY(g.tables.ensure(t.size()));
  CUDA_TRY(cudaMemcpy(g.tables.p, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
  TRY(g.done.ensure(1));
  CUDA_TRY(cudaMemset(g.done.p, 0, sizeof(unsigned int)));
  TRY(g.partials.ensure(2));
  CUDA_TRY(cudaMemset(g.partials.p, 0, 2 * sizeof(uint64_t)));
  TRY(g.result.ensure(2));
  if (!g.h_res) CUDA_TRY(cudaMallocHost(&g.h_res, 2 * sizeof(uint64_t)));
  g.ready = true;
  return 0;
}

// options not set yet (a call may plan before ensure_ready): the defaults
void ensure_options() {
  if (g.opt.segment_kb == 0) default_options(g.opt);
}
size_t seg_bits() {
  ensure_options();
  return (size_t)g.opt.segment_kb * 8192;
}
size_t smem_for(uint32_t segment_kb, uint32_t wheel) {
  return (size_t)segment_kb * 1024 + sv::tables_words(ng_for_wheel(wheel)) * 4 + sv::kSmemAlign;
}
size_t sieve_smem() {
  ensure_options();
  return smem_for(g.opt.segment_kb, g.opt.wheel);
}

int ensure_smem_attr() {
  const size_t sm = sieve_smem();
  if (g.smem_limit_set == sm) return 0;
  CUDA_TRY(sv::set_sieve_smem_limits(sm));
  g.smem_limit_set = sm;
  return 0;
}

// resident sieve CTAs per SM for the current (threads, shared memory), from
// the occupancy query, cached per key and refreshed whenever the key changes
int occupancy() {
  const size_t key = sieve_smem() * 2048 + g.opt.threads;
  if (g.occ_key != key) {
    g.occ = sv::sieve_max_ctas_per_sm(0, 0, (int)g.opt.threads, sieve_smem());
    g.occ_key = key;
  }
  return g.occ > 0 ? g.occ : 1;
}

// Persistent grid: nsm x (resident CTAs per SM).  An explicit ctas_per_sm is
// clamped to the occupancy: every CTA of a launch must be resident (the
// fused A2's grid barriers and the list mode's look-back wait on CTAs of the
// same launch).
int grid_for(uint64_t nseg) {
  if (g.nsm <= 0) return 148;  // before the device is initialised (planning only)
  const int occ = occupancy();
  int per = g.opt.ctas_per_sm > 0 ? std::min((int)g.opt.ctas_per_sm, occ) : occ;
  uint64_t grid = (uint64_t)g.nsm * per;
  if (grid > nseg) grid = nseg;
  return grid < 1 ? 1 : (int)grid;
}

int validate(uint64_t lo, uint64_t hi) {
  if (lo > hi) return fail(SIEVE_EINVAL, "lo (%llu) > hi (%llu)", (unsigned long long)lo,
                           (unsigned long long)hi);
  if (hi > SIEVE_MAX_HI) return fail(SIEVE_ERANGE, "hi (%llu) > 2^48", (unsigned long long)hi);
  return 0;
}

int grid_for(uint64_t nseg);

// Step A1 segment size: the range is cut into w waves of G segments (G the
// persistent grid), w = ceil(B / (S_max G)), with S = ceil(B / (w G)) rounded
// up to a T-layout block (1024 slots): every CTA sieves the same number of
// equal segments (a 2.48-wave launch would otherwise run 3 waves, the last
// half empty; coarser rounding, e.g. to 64 Ki slots, leaves up to w - 1
// segments short of w G and their CTAs idle for a whole segment), and a small
// range still spreads over all SMs.  65536 <= S <= S_max (option segment_kb).
uint64_t balanced_sbits(uint64_t nbits) {
  const uint64_t smax = seg_bits();
  if (nbits == 0) return smax;
  const uint64_t G = (uint64_t)grid_for(~0ull);
  const uint64_t waves = (nbits + smax * G - 1) / (smax * G);
  uint64_t S = (nbits + waves * G - 1) / (waves * G);
#ifndef SIEVE_SROUND
#define SIEVE_SROUND 1024
#endif
  S = (S + SIEVE_SROUND - 1) / SIEVE_SROUND * SIEVE_SROUND;
  return std::min(smax, std::max<uint64_t>(S, 65536));
}

Plan make_plan(uint64_t lo, uint64_t hi) {
  Plan P;
  P.lo = lo;
  P.hi = hi;
  P.o0 = lo | 1;
  P.nbits = hi > lo ? hi / 2 - lo / 2 : 0;
  P.words = (P.nbits + 31) / 32;
  P.sbits = balanced_sbits(P.nbits);
  P.nseg = (P.nbits + P.sbits - 1) / P.sbits;
  P.r = hi >= 2 ? isqrt_u64(hi - 1) : 0;
  P.two = lo <= 2 && 2 < hi;
  return P;
}

int ensure_smem_attr();

uint64_t base_capacity(uint64_t r) {
  // pi(x) < 1.25506 x / ln x for x > 1 (Rosser-Schoenfeld); generous slack
  if (r < 64) return 32;
  const double x = (double)r;
  return (uint64_t)(1.26 * x / std::log(x)) + 64;
}

// K1 into the library's scratch (or the given buffers)
int base_primes(uint64_t r, uint32_t *primes, uint64_t *recips, uint64_t cap, uint32_t *nbase,
                cudaStream_t s) {
  if (r > (1ull << 24)) return fail(SIEVE_ERANGE, "base-prime bound %llu > 2^24", (unsigned long long)r);
  const uint32_t rs = (uint32_t)isqrt_u64(r);
  TRY(ensure_smem_attr());
  const uint32_t ns = sv::base_slices((uint32_t)r);
  if (ns > g.kflags.n) {
    TRY(g.kflags.ensure(ns));
    CUDA_TRY(cudaMemsetAsync(g.kflags.p, 0, g.kflags.n * sizeof(uint64_t), s));
    g.epoch = 0;
  }
  g.epoch = (g.epoch + 1) & 0xFFFF;
  if (g.epoch == 0) {  // 2^16 launches: clear stale tags once
    CUDA_TRY(cudaMemsetAsync(g.kflags.p, 0, g.kflags.n * sizeof(uint64_t), s));
    g.epoch = 1;
  }
  CUDA_TRY(sv::launch_base_primes((uint32_t)r, rs, primes, recips, (uint32_t)cap, nbase,
                                  g.kflags.p ? g.kflags.p : nullptr, g.epoch, g.nsm, g.prof, s));
  g_launches += 1;
  return 0;
}

int own_base(uint64_t r) {
  const uint64_t cap = base_capacity(r);
  TRY(g.primes.ensure(cap));
  TRY(g.recips.ensure(cap));
  TRY(g.nbase.ensure(1));
  return base_primes(r, g.primes.p, g.recips.p, cap, g.nbase.p, g.stream());
}

sv::SieveParams params_for(const Plan &P, const uint32_t *primes, const uint64_t *recips,
                           const uint32_t *nbase, uint64_t *result) {
  sv::SieveParams sp;
  memset(&sp, 0, sizeof sp);
  sp.o0 = P.o0;
  sp.nbits = P.nbits;
  sp.nseg = P.nseg;
  sp.seg_bits = (uint32_t)P.sbits;
  sp.r = (uint32_t)P.r;
  sp.primes = primes;
  sp.recips = recips;
  sp.nbase = nbase;
  sp.tables = g.tables.p;
  sp.add_two = P.two ? 1u : 0u;
  sp.done = g.done.p;
  sp.result = result;
  sp.prof = g.prof;
  sp.flags = g.flags;
  return sp;
}

// Step A5 (option buckets = 1): per-segment buckets for the primes with
// fewer than kBucketHits hits per segment (p > S / kBucketHits), for a range
// sieved in contiguous runs of segments per CTA.  Not in batch mode (one or
// two segments per interval: nothing to skip), when no such prime exists, and
// when a CTA's run exceeds 2^31 odd slots (bucket offsets are 32-bit).
int setup_buckets(sv::SieveParams &sp, int grid) {
  sp.buckets = nullptr;
  if (g.opt.buckets != 1) return 0;
  const uint64_t S = sp.seg_bits;
  if ((uint64_t)sp.r <= S / sv::kBucketHits) return 0;
  const uint64_t run = (sp.nseg + grid - 1) / grid * S;
  if (run >= (1ull << 31)) return 0;
  const uint64_t nw = g.opt.threads / 32;
  const uint64_t capw = (base_capacity(sp.r) + nw - 1) / nw;
  const uint64_t ring = std::min<uint64_t>(sv::kMaxRing, (sp.r + S - 1) / S + 2);
  TRY(g.buckets.ensure((size_t)grid * ring * nw * capw));
  sp.buckets = g.buckets.p;
  sp.ring = (uint32_t)ring;
  sp.capw = (uint32_t)capw;
  sp.inv_seg = (uint32_t)(((1ull << 32) + S - 1) / S);
  return 0;
}

// Where a sieve launch gets its base primes (A2): already in sp.primes
// (req == nullptr), or computed into req's buffers in the same launch (fused
// A2, cooperative) when every CTA's slice of the odd numbers <= r fits its
// segment buffer, else by K1 first.
struct BaseReq {
  uint32_t *primes;
  uint64_t *recips;
  uint32_t *nbase;
  uint64_t cap;
  uint64_t r;
};

// scratch of the fused A2 in the segment buffer (S bits, below the wheel
// tables): small primes and staging, the slice bitmap (L bits) and its
// primes staged for emission (<= L/3 + 2: one of three consecutive odd
// numbers is a multiple of 3)
bool fused_fits(uint64_t r, int grid, uint64_t sbits) {
  if (g.flags & (sv::kFlagNoCoop | sv::kFlagCluster)) return false;  // diagnostics: K1 + an ordinary launch
  if (grid > g.nsm * occupancy()) return false;      // not co-resident (grid_for clamps: never)
  const uint64_t imax = r >= 3 ? (r - 1) / 2 : 0;
  const uint64_t L = ((imax + grid - 1) / grid + 31) / 32 * 32;
  return sv::kMaxSmallWords + 128 + L / 32 + L / 3 + 2 <= sbits / 32;
}

int run_sieve(int mode, sv::SieveParams sp, uint64_t nwork, const BaseReq *req = nullptr) {
  TRY(ensure_smem_attr());
  const int grid = grid_for(nwork);
  sp.partials = g.partials.p;  // [2], zeroed at init, reset by every launch's last CTA
  // not in list mode: its look-back needs the segments of a wave in flight
  // together (round robin), a CTA's contiguous run would serialise it
  if (mode == sv::kCount || mode == sv::kBitmap) TRY(setup_buckets(sp, grid));
  const int ng = ng_for_wheel(g.opt.wheel);
  // the kPlain kernels (launch_t: default wheel, r > S / kPlainHits) read the
  // plain primes as {p, floor(2^44/p)} (written by the fused A2, else by k_pack44)
  bool pack = false;
  if (SIEVE_PACK44 && SIEVE_COUNT_PLAIN && mode != sv::kBatch && ng == SIEVE_PLAIN_NG &&
      (uint64_t)sp.r > sp.seg_bits / SIEVE_PLAIN_HITS) {
    TRY(g.pk44.ensure(base_capacity(sp.r)));
    sp.pk44 = g.pk44.p;
    pack = true;
  }
  if (req) {
    sp.primes = req->primes;
    sp.recips = req->recips;
    sp.nbase = req->nbase;
    if (fused_fits(req->r, grid, sp.seg_bits)) {
      if (!g.gbar.p) {
        TRY(g.gbar.ensure(1));
        CUDA_TRY(cudaMemsetAsync(g.gbar.p, 0, sizeof(unsigned int), g.stream()));
      }
      TRY(g.bcounts.ensure((size_t)grid + 7));  // counts, then the region boundaries
      sv::SieveParams fp = sp;
      fp.bprimes = req->primes;
      fp.brecips = req->recips;
      fp.bnbase = req->nbase;
      fp.bcap = (uint32_t)std::min<uint64_t>(req->cap, 0xFFFFFFFFull);
      fp.rs = (uint32_t)isqrt_u64(req->r);
      fp.bcounts = g.bcounts.p;
      fp.gbar = g.gbar.p;
      const cudaError_t e = sv::launch_sieve(ng, mode, fp, grid, (int)g.opt.threads, sieve_smem(), g.stream());
      if (e == cudaSuccess) {
        g_launches += 1;
        return 0;
      }
      // the cooperative launch was refused (e.g. not every CTA can be
      // resident under MPS or a co-tenant): nothing ran; clear the
      // (non-sticky) launch error and take the K1 + ordinary-launch path
      cudaGetLastError();
      g_coop_fallbacks += 1;
    }
    TRY(base_primes(req->r, req->primes, req->recips, req->cap, req->nbase, g.stream()));
  }
  if (mode == sv::kCount && (g.flags & sv::kFlagCluster) && !sp.peers && !sp.buckets && grid >= 2) {
    // F3 diagnostics: the cluster-pair kernel (two CTAs per super-segment)
    CUDA_TRY(sv::launch_sieve_cluster(ng, sp, grid, (int)g.opt.threads, sieve_smem(), g.stream()));
    g_launches += 1;
    return 0;
  }
  if (pack) {
    CUDA_TRY(sv::launch_pack44(sp.primes, sp.recips, sp.nbase, sp.pk44, (uint32_t)base_capacity(sp.r),
                               g.stream()));
    g_launches += 1;
  }
  CUDA_TRY(sv::launch_sieve(ng, mode, sp, grid, (int)g.opt.threads, sieve_smem(), g.stream()));
  g_launches += 1;
  return 0;
}

// count/sum of [lo, hi) into device result[0..1]; empty/odd-free ranges handled
int stats_async(const Plan &P, const uint32_t *primes, const uint64_t *recips, const uint32_t *nbase,
                uint64_t *result, const BaseReq *req = nullptr) {
  if (P.nbits == 0) {
    if (req) TRY(base_primes(req->r, req->primes, req->recips, req->cap, req->nbase, g.stream()));
    uint64_t h[2] = {P.two ? 1ull : 0ull, P.two ? 2ull : 0ull};
    CUDA_TRY(cudaMemcpyAsync(result, h, sizeof h, cudaMemcpyHostToDevice, g.stream()));
    CUDA_TRY(cudaStreamSynchronize(g.stream()));  // h is on this stack frame
    return 0;
  }
  sv::SieveParams sp = params_for(P, primes, recips, nbase, result);
  return run_sieve(sv::kCount, sp, P.nseg, req);
}

int bitmap_async(const Plan &P, const uint32_t *primes, const uint64_t *recips, const uint32_t *nbase,
                 uint32_t *out, uint64_t *result, const BaseReq *req, bool want_sum) {
  if (P.nbits == 0) return stats_async(P, primes, recips, nbase, result, req);
  sv::SieveParams sp = params_for(P, primes, recips, nbase, result);
  if (!want_sum) sp.flags |= sv::kFlagNoSum;
  sp.out = out;
  sp.out_words = P.words;
  sp.out_vec4 = ((uintptr_t)out & 15u) == 0 ? 1u : 0u;
  return run_sieve(sv::kBitmap, sp, P.nseg, req);
}

// the library's own base-prime buffers, sized for r, as a fused-A2 request
int own_req(uint64_t r, BaseReq &q) {
  const uint64_t cap = base_capacity(r);
  TRY(g.primes.ensure(cap));
  TRY(g.recips.ensure(cap));
  TRY(g.nbase.ensure(1));
  q = BaseReq{g.primes.p, g.recips.p, g.nbase.p, cap, r};
  return 0;
}

// F4: count/sum of this rank's [lo, hi) summed over every attached rank, the
// all-reduce done inside the sieve kernel's last CTA (peer.cuh)
int stats_allreduce_async(const Plan &P, const uint32_t *primes, const uint64_t *recips,
                          const uint32_t *nbase, uint64_t *result, const BaseReq *req = nullptr) {
  auto &pe = g.peer;
  pe.epoch += 1;
  if (P.nbits == 0) {  // no sieve launch: publish (0, 0) or (1, 2) alone
    if (req) TRY(base_primes(req->r, req->primes, req->recips, req->cap, req->nbase, g.stream()));
    CUDA_TRY(sv::launch_peer_only(pe.ptrs.p, pe.world, pe.rank, pe.epoch, pe.timeout_ns,
                                  P.two ? 1 : 0, P.two ? 2 : 0, result, g.stream()));
    g_launches += 1;
    return 0;
  }
  sv::SieveParams sp = params_for(P, primes, recips, nbase, result);
  sp.peers = pe.ptrs.p;
  sp.pepoch = pe.epoch;
  sp.timeout_ns = pe.timeout_ns;
  sp.world = pe.world;
  sp.rank = pe.rank;
  return run_sieve(sv::kCount, sp, P.nseg, req);
}

void peer_detach() {
  for (void *q : g.peer.opened)
    if (q) cudaIpcCloseMemHandle(q);
  g.peer.opened.clear();
  g.peer.world = 0;
  g.peer.rank = 0;
}

int peer_attach(unsigned long long *const *slabs, uint32_t world, uint32_t rank,
                uint32_t timeout_ms) {
  TRY(g.peer.ptrs.ensure(world));
  CUDA_TRY(cudaMemcpy(g.peer.ptrs.p, slabs, world * sizeof(void *), cudaMemcpyHostToDevice));
  g.peer.world = world;
  g.peer.rank = rank;
  g.peer.epoch = 0;
  g.peer.timeout_ns = (uint64_t)(timeout_ms ? timeout_ms : 10000) * 1000000ull;
  return 0;
}

bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int fetch_result(uint64_t *count, uint64_t *sum) {
  CUDA_TRY(cudaMemcpyAsync(g.h_res, g.result.p, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                           g.stream()));
  CUDA_TRY(cudaStreamSynchronize(g.stream()));
  if (count) *count = g.h_res[0];
  if (sum) *sum = g.h_res[1];
  return 0;
}

int do_stats(uint64_t lo, uint64_t hi, uint64_t *count, uint64_t *sum) {
  TRY(validate(lo, hi));
  TRY(ensure_ready());
  const Plan P = make_plan(lo, hi);
  if (P.nbits == 0) {
    if (count) *count = P.two ? 1 : 0;
    if (sum) *sum = P.two ? 2 : 0;
    return 0;
  }
  BaseReq q;
  TRY(own_req(P.r, q));
  TRY(stats_async(P, q.primes, q.recips, q.nbase, g.result.p, &q));
  return fetch_result(count, sum);
}

int64_t do_bitmap(uint64_t lo, uint64_t hi, uint32_t *out) {
  TRY(validate(lo, hi));
  const Plan P0 = make_plan(lo, hi);
  if (P0.words > 0 && !out) return fail(SIEVE_EINVAL, "out is NULL for %llu words", (unsigned long long)P0.words);
  TRY(ensure_ready());
  const Plan P = make_plan(lo, hi);
  if (P.nbits == 0) return P.two ? 1 : 0;
  BaseReq q;
  TRY(own_req(P.r, q));
  const bool dev = is_device_ptr(out);
  uint32_t *dst = out;
  if (!dev) {
    TRY(g.bitmap.ensure(P.words));
    dst = g.bitmap.p;
  }
  TRY(bitmap_async(P, q.primes, q.recips, q.nbase, dst, g.result.p, &q, false));
  if (!dev)
    CUDA_TRY(cudaMemcpyAsync(out, dst, P.words * 4, cudaMemcpyDeviceToHost, g.stream()));
  uint64_t c = 0;
  TRY(fetch_result(&c, nullptr));
  return (int64_t)c;
}

int64_t do_primes(uint64_t lo, uint64_t hi, uint64_t *out, uint64_t cap) {
  TRY(validate(lo, hi));
  if (cap > 0 && !out) return fail(SIEVE_EINVAL, "out is NULL with cap %llu", (unsigned long long)cap);
  TRY(ensure_ready());
  const Plan P = make_plan(lo, hi);
  if (P.nbits == 0) {
    if (P.two && cap > 0) {
      const uint64_t two = 2;
      if (is_device_ptr(out)) {
        CUDA_TRY(cudaMemcpyAsync(out, &two, 8, cudaMemcpyHostToDevice, g.stream()));
        CUDA_TRY(cudaStreamSynchronize(g.stream()));
      } else {
        out[0] = 2;
      }
    }
    return P.two ? 1 : 0;
  }
  BaseReq q;
  TRY(own_req(P.r, q));
  if (cap == 0) {  // size query: count mode
    TRY(stats_async(P, q.primes, q.recips, q.nbase, g.result.p, &q));
  } else {
    const bool dev = is_device_ptr(out);
    uint64_t *dst = out;
    if (!dev) {
      TRY(g.list.ensure(cap));
      dst = g.list.p;
    }
    // list mode: one sieve launch writes the list (decoupled look-back)
    if (P.nseg > g.lflags.n) {
      TRY(g.lflags.ensure(P.nseg));
      CUDA_TRY(cudaMemsetAsync(g.lflags.p, 0, g.lflags.n * sizeof(unsigned long long), g.stream()));
      g.lepoch = 0;
    }
    g.lepoch = (g.lepoch + 1) & 0xFFFF;
    if (g.lepoch == 0) {  // 2^16 launches: clear stale tags once
      CUDA_TRY(cudaMemsetAsync(g.lflags.p, 0, g.lflags.n * sizeof(unsigned long long), g.stream()));
      g.lepoch = 1;
    }
    sv::SieveParams sp = params_for(P, g.primes.p, g.recips.p, g.nbase.p, g.result.p);
    sp.list = dst;
    sp.list_cap = cap;
    sp.lflags = g.lflags.p;
    sp.lepoch = g.lepoch;
    TRY(run_sieve(sv::kList, sp, P.nseg, &q));
    uint64_t c = 0;
    TRY(fetch_result(&c, nullptr));
    if (!dev) {
      const uint64_t n = std::min(c, cap);
      CUDA_TRY(cudaMemcpyAsync(out, dst, n * 8, cudaMemcpyDeviceToHost, g.stream()));
      CUDA_TRY(cudaStreamSynchronize(g.stream()));
    }
    return (int64_t)c;
  }
  uint64_t c = 0;
  TRY(fetch_result(&c, nullptr));
  return (int64_t)c;
}

// Step A10 on device-resident intervals: base primes <= isqrt(hi_max - 1)
// (K1), the plan on the device (launch_batch_plan: items of <= S odd slots,
// largest cost class first), then the batch sieve over the planned items.
// result: [2 n] (count, sum mod 2^64) per interval, overwritten.
int batch_async(const uint64_t *lo, const uint64_t *hi, uint64_t n, uint64_t hi_max,
                uint64_t width_max, uint64_t *result) {
  if (n == 0) return 0;
  if (n > 0xFFFFFFFFull) return fail(SIEVE_EINVAL, "n = %llu intervals > 2^32 - 1", (unsigned long long)n);
  if (hi_max > SIEVE_MAX_HI) return fail(SIEVE_ERANGE, "hi_max > 2^48");
  const uint64_t S = seg_bits();
  const uint64_t kcap = (width_max / 2 + 1 + S - 1) / S + 1;  // items of one interval, at most
  if (n * kcap > 0xFFFFFFFFull) return fail(SIEVE_EINVAL, "too many batch items");
  const uint64_t rmax = hi_max >= 2 ? isqrt_u64(hi_max - 1) : 0;
  TRY(own_base(rmax));
  const uint64_t bcap = base_capacity(rmax);
  TRY(g.pk44.ensure(bcap));
  CUDA_TRY(sv::launch_pack44(g.primes.p, g.recips.p, g.nbase.p, g.pk44.p, (uint32_t)bcap, g.stream()));
  g_launches += 1;
  if (!g.plan.p) {
    TRY(g.plan.ensure(2 * sv::kPlanBuckets));
    CUDA_TRY(cudaMemsetAsync(g.plan.p, 0, 2 * sv::kPlanBuckets * sizeof(uint32_t), g.stream()));
  }
  TRY(g.nitems.ensure(1));
  TRY(g.items.ensure(n * kcap));
  CUDA_TRY(sv::launch_batch_plan(lo, hi, n, (uint32_t)S, width_max, g.primes.p, g.nbase.p,
                                 g.plan.p, g.items.p, g.nitems.p, result, g.stream()));
  g_launches += 3;
  Plan dummy = make_plan(0, 0);
  sv::SieveParams sp = params_for(dummy, g.primes.p, g.recips.p, g.nbase.p, result);
  sp.items = g.items.p;
  sp.nitems = g.nitems.p;
  sp.pk44 = SIEVE_PACK44 ? g.pk44.p : nullptr;
  sp.nseg = n * kcap;  // bound for the grid size; the kernel reads *nitems
  sp.r = (uint32_t)rmax;
  return run_sieve(sv::kBatch, sp, n * kcap);
}

int do_batch(const uint64_t *lo, const uint64_t *hi, uint64_t n, uint64_t *count, uint64_t *sum) {
  if (n == 0) return 0;
  if (!lo || !hi || !count || !sum) return fail(SIEVE_EINVAL, "NULL array in sieve_batch");
  uint64_t hi_max = 0, width_max = 0;
  for (uint64_t i = 0; i < n; ++i) {
    TRY(validate(lo[i], hi[i]));
    hi_max = std::max(hi_max, hi[i]);
    width_max = std::max(width_max, hi[i] - lo[i]);
  }
  TRY(ensure_ready());
  // the intervals to the device, the plan and the sieve there, the results back
  TRY(g.blo.ensure(n));
  TRY(g.bhi.ensure(n));
  TRY(g.bres.ensure(2 * n));
  CUDA_TRY(cudaMemcpyAsync(g.blo.p, lo, n * 8, cudaMemcpyHostToDevice, g.stream()));
  CUDA_TRY(cudaMemcpyAsync(g.bhi.p, hi, n * 8, cudaMemcpyHostToDevice, g.stream()));
  TRY(batch_async(g.blo.p, g.bhi.p, n, hi_max, width_max, g.bres.p));
  std::vector<uint64_t> h(2 * n);
  CUDA_TRY(cudaMemcpyAsync(h.data(), g.bres.p, 2 * n * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                           g.stream()));
  CUDA_TRY(cudaStreamSynchronize(g.stream()));
  for (uint64_t i = 0; i < n; ++i) {
    count[i] = h[2 * i];
    sum[i] = h[2 * i + 1];
  }
  return 0;
}

// Step F2 calls: all pointers of a call on the device (used in place) or all
// on the host (staged through device scratch).  Returns 0 or an error code.
struct Staged {
  DevBuf<uint8_t> buf;
};
Staged g_f2;

int f2_run(const void *const *in, const size_t *in_bytes, int nin, void *out, size_t out_bytes,
           int (*launch)(void *const *dev_in, void *dev_out, cudaStream_t s)) {
  bool any_dev = false, any_host = false;
  for (int k = 0; k < nin; ++k) (is_device_ptr(in[k]) ? any_dev : any_host) = true;
  (is_device_ptr(out) ? any_dev : any_host) = true;
  if (any_dev && any_host) return fail(SIEVE_EINVAL, "mixed host and device pointers");
  if (any_dev) {
    void *dev_in[4];
    for (int k = 0; k < nin; ++k) dev_in[k] = const_cast<void *>(in[k]);
    TRY(launch(dev_in, out, g.stream()));
    CUDA_TRY(cudaStreamSynchronize(g.stream()));
    return 0;
  }
  size_t total = out_bytes;
  size_t off[4];
  for (int k = 0; k < nin; ++k) {
    off[k] = (total + 15) / 16 * 16;
    total = off[k] + in_bytes[k];
  }
  TRY(g_f2.buf.ensure(total + 16));
  uint8_t *base = g_f2.buf.p;
  void *dev_in[4];
  for (int k = 0; k < nin; ++k) {
    dev_in[k] = base + off[k];
    CUDA_TRY(cudaMemcpyAsync(dev_in[k], in[k], in_bytes[k], cudaMemcpyHostToDevice, g.stream()));
  }
  TRY(launch(dev_in, base, g.stream()));
  CUDA_TRY(cudaMemcpyAsync(out, base, out_bytes, cudaMemcpyDeviceToHost, g.stream()));
  CUDA_TRY(cudaStreamSynchronize(g.stream()));
  return 0;
}

uint64_t f2_n = 0;
uint32_t f2_iters = 0;

int launch_modpow_cb(void *const *d, void *o, cudaStream_t s) {
  CUDA_TRY(sv::launch_modpow((const uint64_t *)d[0], (const uint64_t *)d[1], (const uint64_t *)d[2],
                             f2_n, (uint64_t *)o, s));
  g_launches += 1;
  return 0;
}
int launch_fermat_cb(void *const *d, void *o, cudaStream_t s) {
  CUDA_TRY(sv::launch_fermat((const uint64_t *)d[0], f2_n, (const uint64_t *)d[1], f2_iters,
                             (uint8_t *)o, s));
  g_launches += 1;
  return 0;
}
int launch_is_prime_cb(void *const *d, void *o, cudaStream_t s) {
  CUDA_TRY(sv::launch_is_prime((const uint64_t *)d[0], f2_n, (uint8_t *)o, s));
  g_launches += 1;
  return 0;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

int64_t sieve_count(uint64_t lo, uint64_t hi) {
  std::lock_guard<std::mutex> lk(g.mu);
  uint64_t c = 0;
  TRY(do_stats(lo, hi, &c, nullptr));
  return (int64_t)c;
}

int64_t sieve_bitmap(uint64_t lo, uint64_t hi, uint32_t *out) {
  std::lock_guard<std::mutex> lk(g.mu);
  return do_bitmap(lo, hi, out);
}

int64_t sieve_primes(uint64_t lo, uint64_t hi, uint64_t *out, uint64_t cap) {
  std::lock_guard<std::mutex> lk(g.mu);
  return do_primes(lo, hi, out, cap);
}

uint64_t sieve_bitmap_words(uint64_t lo, uint64_t hi) {
  if (hi <= lo) return 0;
  return (hi / 2 - lo / 2 + 31) / 32;
}

int sieve_stats(uint64_t lo, uint64_t hi, uint64_t *count, uint64_t *sum_mod_2_64) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (!count || !sum_mod_2_64) return fail(SIEVE_EINVAL, "NULL output in sieve_stats");
  return do_stats(lo, hi, count, sum_mod_2_64);
}

int sieve_batch(const uint64_t *lo, const uint64_t *hi, uint64_t n, uint64_t *count,
                uint64_t *sum_mod_2_64) {
  std::lock_guard<std::mutex> lk(g.mu);
  return do_batch(lo, hi, n, count, sum_mod_2_64);
}

int sieve_batch_async(const uint64_t *lo, const uint64_t *hi, uint64_t n, uint64_t hi_max,
                      uint64_t width_max, uint64_t *result) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (n == 0) return 0;
  if (!lo || !hi || !result) return fail(SIEVE_EINVAL, "NULL array in sieve_batch_async");
  TRY(ensure_ready());
  return batch_async(lo, hi, n, hi_max, width_max, result);
}

uint64_t sieve_base_capacity(uint64_t r) { return base_capacity(r); }

int sieve_base_primes_async(uint64_t r, uint32_t *primes, uint64_t *recips, uint64_t cap,
                            uint32_t *nbase) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (!primes || !recips || !nbase) return fail(SIEVE_EINVAL, "NULL buffer");
  if (cap < base_capacity(r)) return fail(SIEVE_EINVAL, "cap %llu < sieve_base_capacity(%llu)",
                                          (unsigned long long)cap, (unsigned long long)r);
  TRY(ensure_ready());
  return base_primes(r, primes, recips, cap, nbase, g.stream());
}

int sieve_prepare_base_async(const uint32_t *primes, const uint32_t *nbase, uint64_t *recips,
                             uint64_t cap) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (!primes || !recips || !nbase) return fail(SIEVE_EINVAL, "NULL buffer");
  TRY(ensure_ready());
  CUDA_TRY(sv::launch_prepare(primes, nbase, recips, (uint32_t)cap, g.stream()));
  g_launches += 1;
  return 0;
}

int sieve_stats_async(uint64_t lo, uint64_t hi, const uint32_t *primes, const uint64_t *recips,
                      const uint32_t *nbase, uint64_t *result) {
  std::lock_guard<std::mutex> lk(g.mu);
  TRY(validate(lo, hi));
  if (!primes || !recips || !nbase || !result) return fail(SIEVE_EINVAL, "NULL buffer");
  TRY(ensure_ready());
  return stats_async(make_plan(lo, hi), primes, recips, nbase, result);
}

int sieve_stats_base_async(uint64_t lo, uint64_t hi, uint32_t *primes, uint64_t *recips,
                           uint32_t *nbase, uint64_t cap, int allreduce, uint64_t *result) {
  std::lock_guard<std::mutex> lk(g.mu);
  TRY(validate(lo, hi));
  if (!primes || !recips || !nbase || !result) return fail(SIEVE_EINVAL, "NULL buffer");
  const Plan P = make_plan(lo, hi);
  if (cap < base_capacity(P.r)) return fail(SIEVE_EINVAL, "cap %llu < sieve_base_capacity(%llu)",
                                            (unsigned long long)cap, (unsigned long long)P.r);
  if (allreduce && g.peer.world == 0) return fail(SIEVE_EINVAL, "no peers attached (sieve_peer_attach)");
  TRY(ensure_ready());
  const BaseReq q{primes, recips, nbase, cap, P.r};
  if (allreduce) return stats_allreduce_async(P, primes, recips, nbase, result, &q);
  return stats_async(P, primes, recips, nbase, result, &q);
}

int sieve_bitmap_async(uint64_t lo, uint64_t hi, const uint32_t *primes, const uint64_t *recips,
                       const uint32_t *nbase, uint32_t *out, uint64_t *result) {
  std::lock_guard<std::mutex> lk(g.mu);
  TRY(validate(lo, hi));
  if (!primes || !recips || !nbase || !result) return fail(SIEVE_EINVAL, "NULL buffer");
  const Plan P = make_plan(lo, hi);
  if (P.words && !out) return fail(SIEVE_EINVAL, "NULL out");
  TRY(ensure_ready());
  return bitmap_async(P, primes, recips, nbase, out, result, nullptr, !g.opt.bitmap_count_only);
}

int sieve_bitmap_base_async(uint64_t lo, uint64_t hi, uint32_t *primes, uint64_t *recips,
                            uint32_t *nbase, uint64_t cap, uint32_t *out, uint64_t *result) {
  std::lock_guard<std::mutex> lk(g.mu);
  TRY(validate(lo, hi));
  if (!primes || !recips || !nbase || !result) return fail(SIEVE_EINVAL, "NULL buffer");
  const Plan P = make_plan(lo, hi);
  if (P.words && !out) return fail(SIEVE_EINVAL, "NULL out");
  if (cap < base_capacity(P.r)) return fail(SIEVE_EINVAL, "cap %llu < sieve_base_capacity(%llu)",
                                            (unsigned long long)cap, (unsigned long long)P.r);
  TRY(ensure_ready());
  const BaseReq q{primes, recips, nbase, cap, P.r};
  return bitmap_async(P, primes, recips, nbase, out, result, &q, !g.opt.bitmap_count_only);
}

int sieve_peer_slab_handle(void *handle_out) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (!handle_out) return fail(SIEVE_EINVAL, "NULL handle_out");
  TRY(ensure_ready());
  if (!g.peer.slab) {
    CUDA_TRY(cudaMalloc(&g.peer.slab, sv::kPeerSlabBytes));
    CUDA_TRY(cudaMemset(g.peer.slab, 0, sv::kPeerSlabBytes));
  }
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, g.peer.slab));
  static_assert(sizeof h == SIEVE_IPC_HANDLE_BYTES, "cudaIpcMemHandle_t size");
  memcpy(handle_out, &h, sizeof h);
  return 0;
}

int sieve_peer_attach(const void *handles, int world, int rank, uint32_t timeout_ms) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (!handles) return fail(SIEVE_EINVAL, "NULL handles");
  if (world < 1 || world > SIEVE_MAX_PEERS || rank < 0 || rank >= world)
    return fail(SIEVE_EINVAL, "world %d / rank %d out of range (1 <= world <= %d)", world, rank,
                SIEVE_MAX_PEERS);
  TRY(ensure_ready());
  if (!g.peer.slab) return fail(SIEVE_EINVAL, "sieve_peer_slab_handle was not called");
  CUDA_TRY(cudaStreamSynchronize(g.stream()));
  peer_detach();
  std::vector<unsigned long long *> slabs(world, nullptr);
  for (int q = 0; q < world; ++q) {
    if (q == rank) {
      slabs[q] = g.peer.slab;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char *)handles + (size_t)q * SIEVE_IPC_HANDLE_BYTES, sizeof h);
    void *ptr = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      peer_detach();
      return fail(SIEVE_ECUDA, "cudaIpcOpenMemHandle(rank %d) failed: %s", q, cudaGetErrorString(e));
    }
    g.peer.opened.push_back(ptr);
    slabs[q] = (unsigned long long *)ptr;
  }
  // stale epochs of an earlier attach must not match the new ones
  CUDA_TRY(cudaMemset(g.peer.slab, 0, sv::kPeerSlabBytes));
  return peer_attach(slabs.data(), (uint32_t)world, (uint32_t)rank, timeout_ms);
}

int sieve_peer_attach_ptrs(void *const *slabs, int world, int rank, uint32_t timeout_ms) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (!slabs) return fail(SIEVE_EINVAL, "NULL slabs");
  if (world < 1 || world > SIEVE_MAX_PEERS || rank < 0 || rank >= world)
    return fail(SIEVE_EINVAL, "world %d / rank %d out of range (1 <= world <= %d)", world, rank,
                SIEVE_MAX_PEERS);
  for (int q = 0; q < world; ++q)
    if (!slabs[q]) return fail(SIEVE_EINVAL, "NULL slab for rank %d", q);
  TRY(ensure_ready());
  CUDA_TRY(cudaStreamSynchronize(g.stream()));
  peer_detach();
  return peer_attach((unsigned long long *const *)slabs, (uint32_t)world, (uint32_t)rank,
                     timeout_ms);
}

int sieve_peer_detach(void) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.ready) CUDA_TRY(cudaStreamSynchronize(g.stream()));
  peer_detach();
  return 0;
}

uint64_t sieve_peer_epoch(void) { return g.peer.epoch; }

int sieve_stats_allreduce_async(uint64_t lo, uint64_t hi, const uint32_t *primes,
                                const uint64_t *recips, const uint32_t *nbase, uint64_t *result) {
  std::lock_guard<std::mutex> lk(g.mu);
  TRY(validate(lo, hi));
  if (!primes || !recips || !nbase || !result) return fail(SIEVE_EINVAL, "NULL buffer");
  if (g.peer.world == 0) return fail(SIEVE_EINVAL, "no peers attached (sieve_peer_attach)");
  TRY(ensure_ready());
  return stats_allreduce_async(make_plan(lo, hi), primes, recips, nbase, result);
}

int sieve_peer_publish_async(uint64_t count, uint64_t sum) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.peer.world == 0) return fail(SIEVE_EINVAL, "no peers attached (sieve_peer_attach)");
  TRY(ensure_ready());
  auto &pe = g.peer;
  pe.epoch += 1;
  TRY(g.result.ensure(2));
  CUDA_TRY(sv::launch_peer_only(pe.ptrs.p, pe.world, pe.rank, pe.epoch, pe.timeout_ns, count, sum,
                                g.result.p, g.stream(), /*wait=*/false));
  g_launches += 1;
  return 0;
}

int sieve_set_device(int ordinal) {
  std::lock_guard<std::mutex> lk(g.mu);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0)
    return fail(SIEVE_ENODEV, "no CUDA device available");
  if (ordinal < 0 || ordinal >= ndev) return fail(SIEVE_EINVAL, "device %d out of range", ordinal);
  if (g.ready && ordinal != g.device)
    return fail(SIEVE_EINVAL, "device already initialised as %d; call sieve_shutdown first", g.device);
  g.device = ordinal;
  CUDA_TRY(cudaSetDevice(ordinal));
  return 0;
}

int sieve_set_stream(void *cuda_stream) {
  std::lock_guard<std::mutex> lk(g.mu);
  const cudaStream_t next = cuda_stream ? (cudaStream_t)cuda_stream : g.own;
  if (g.ready && next != g.stream()) {
    // every launch shares the library's scratch (partials, tickets, grid
    // barrier, look-back flags, result): work on the new stream starts only
    // after the work already queued on the old one
    cudaEvent_t ev;
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    cudaError_t e = cudaEventRecord(ev, g.stream());
    if (e == cudaSuccess) e = cudaStreamWaitEvent(next, ev, 0);
    cudaEventDestroy(ev);
    CUDA_TRY(e);
  }
  g.user = (cudaStream_t)cuda_stream;
  g.user_set = cuda_stream != nullptr;
  return 0;
}

void *sieve_get_stream(void) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (ensure_ready() < 0) return nullptr;
  return (void *)g.stream();
}

int sieve_set_options(const sieve_options *o) {
  std::lock_guard<std::mutex> lk(g.mu);
  sieve_options n;
  default_options(n);
  if (o) {
    for (int i = 0; i < 2; ++i)
      if (o->reserved[i]) return fail(SIEVE_EINVAL, "reserved option fields must be zero");
    if (o->bitmap_count_only > 1)
      return fail(SIEVE_EINVAL, "bitmap_count_only %u not in {0, 1}", o->bitmap_count_only);
    n.bitmap_count_only = o->bitmap_count_only;
    if (o->buckets > 1) return fail(SIEVE_EINVAL, "buckets %u not in {0, 1}", o->buckets);
    n.buckets = o->buckets;
    if (o->segment_kb) {
      if (o->segment_kb < 4 || o->segment_kb > 224)
        return fail(SIEVE_EINVAL, "segment_kb %u is not in [4, 224]", o->segment_kb);
      n.segment_kb = o->segment_kb;
    }
    if (o->wheel) {
      if (ng_for_wheel(o->wheel) < 0)
        return fail(SIEVE_EINVAL, "wheel %u not in {11,17,23,31,41,47}", o->wheel);
      n.wheel = o->wheel;
    }
    if (o->threads) {
      if (o->threads % 64 != 0 || o->threads < 256 || o->threads > SIEVE_MAX_THREADS)
        return fail(SIEVE_EINVAL, "threads %u is not a multiple of 64 in [256, %d]", o->threads,
                    SIEVE_MAX_THREADS);
      n.threads = o->threads;
    }
    if (o->ctas_per_sm > 32) return fail(SIEVE_EINVAL, "ctas_per_sm %u > 32", o->ctas_per_sm);
    if (smem_for(n.segment_kb, n.wheel) > kMaxDynSmem)
      return fail(SIEVE_EINVAL, "segment_kb %u with wheel %u needs %zu bytes of shared memory (> %zu)",
                  n.segment_kb, n.wheel, smem_for(n.segment_kb, n.wheel), kMaxDynSmem);
    n.ctas_per_sm = o->ctas_per_sm;
  }
  g.opt = n;
  return 0;
}

int sieve_get_options(sieve_options *o) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (!o) return fail(SIEVE_EINVAL, "NULL");
  if (g.opt.segment_kb == 0) default_options(g.opt);
  *o = g.opt;
  return 0;
}

const char *sieve_last_error(void) { return g_err.c_str(); }

void sieve_shutdown(void) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (!g.ready) return;
  cudaStreamSynchronize(g.stream());
  g.tables.release(); g.primes.release(); g.recips.release(); g.pk44.release(); g.nbase.release();
  g.partials.release(); g.done.release(); g.result.release(); g.bitmap.release();
  g.list.release(); g.items.release(); g.bres.release();
  g.blo.release(); g.bhi.release(); g.plan.release(); g.nitems.release();
  g.buckets.release(); g.kflags.release(); g.lflags.release(); g_f2.buf.release();
  g.gbar.release(); g.bcounts.release();  // fused A2 (re-created, zeroed, on demand)
  peer_detach();
  g.peer.ptrs.release();
  if (g.peer.slab) cudaFree(g.peer.slab);
  g.peer.slab = nullptr;
  if (g.h_res) cudaFreeHost(g.h_res);
  g.h_res = nullptr;
  if (g.own) cudaStreamDestroy(g.own);
  g.own = nullptr;
  g.smem_limit_set = 0;
  g.occ_key = 0;
  g.ready = false;
}

uint64_t sieve_kernel_launches(void) { return g_launches.load(); }

int sieve_modpow(const uint64_t *a, const uint64_t *b, const uint64_t *c, uint64_t n, uint64_t *out) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (n == 0) return 0;
  if (!a || !b || !c || !out) return fail(SIEVE_EINVAL, "NULL array in sieve_modpow");
  TRY(ensure_ready());
  f2_n = n;
  const void *in[3] = {a, b, c};
  const size_t by[3] = {n * 8, n * 8, n * 8};
  return f2_run(in, by, 3, out, n * 8, launch_modpow_cb);
}

int sieve_fermat(const uint64_t *p, uint64_t n, const uint64_t *draws, uint32_t iterations,
                 uint8_t *out) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (n == 0) return 0;
  if (iterations == 0) return fail(SIEVE_EINVAL, "iterations must be >= 1 (SPEC.md fermat_test)");
  if (!p || !draws || !out) return fail(SIEVE_EINVAL, "NULL array in sieve_fermat");
  TRY(ensure_ready());
  f2_n = n;
  f2_iters = iterations;
  const void *in[2] = {p, draws};
  const size_t by[2] = {n * 8, n * (size_t)iterations * 8};
  return f2_run(in, by, 2, out, n, launch_fermat_cb);
}

int sieve_is_prime(const uint64_t *nums, uint64_t n, uint8_t *out) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (n == 0) return 0;
  if (!nums || !out) return fail(SIEVE_EINVAL, "NULL array in sieve_is_prime");
  TRY(ensure_ready());
  f2_n = n;
  const void *in[1] = {nums};
  const size_t by[1] = {n * 8};
  return f2_run(in, by, 1, out, n, launch_is_prime_cb);
}

int sieve_debug_set_flags(uint32_t flags) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (flags & ~(sv::kFlagSkipMarking | sv::kFlagSkipA | sv::kFlagSkipB | sv::kFlagSkipC |
                sv::kFlagReverse | sv::kFlagNoCoop | sv::kFlagCluster | sv::kFlagSkipWheel))
    return fail(SIEVE_EINVAL, "unknown debug flags %u", flags);
  g.flags = flags;
  return 0;
}

int sieve_debug_violations(uint64_t *out, int reset) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (!out) return fail(SIEVE_EINVAL, "NULL out");
  TRY(ensure_ready());
  CUDA_TRY(cudaStreamSynchronize(g.stream()));
  unsigned long long v[sv::kVioClasses];
  CUDA_TRY(sv::read_violations(v, reset != 0));
  for (int k = 0; k < sv::kVioClasses; ++k) out[k] = v[k];
  return SIEVE_CHECK_BOUNDS;
}

int sieve_debug_k0(double *lanes_per_clk_per_sm, double *sm_ghz) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (!lanes_per_clk_per_sm || !sm_ghz) return fail(SIEVE_EINVAL, "NULL output");
  TRY(ensure_ready());
  CUDA_TRY(cudaStreamSynchronize(g.stream()));
  CUDA_TRY(sv::k0_smem_atomic_rate(g.nsm, lanes_per_clk_per_sm, sm_ghz));
  g_launches += 3;
  return 0;
}

uint64_t sieve_debug_coop_fallbacks(void) { return g_coop_fallbacks.load(); }

int sieve_debug_set_profile(uint64_t *dev_counters) {
  std::lock_guard<std::mutex> lk(g.mu);
  g.prof = reinterpret_cast<unsigned long long *>(dev_counters);
  return 0;
}

}  // extern "C"
