// pmh_capi.cu -- extern "C" boundary of libpmh.so (declared in include/pmh.h).
//
// Host responsibilities: argument validation with the reference's error
// domain (sketch.py:96-114), per-(device, m) constant tables computed with the
// host glibc exactly as the reference computes them inside each call
// (K:418-420, K:458-459, K:497-498, K:568-579), kernel dispatch, and mapping
// device error flags to the reference's exceptions (errors.py).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/pmh.h"
#include "pmh_pminhash.cuh"
#include "pmh_kernel.cuh"
#include "pmh_flat.cuh"
#include "pmh_join.cuh"
#include "pmh_order.cuh"
#include "pmh_probe.cuh"
#include "pmh_baselines.cuh"
#include "pmh_harness.cuh"
#include "pmh_ingest.h"

#ifndef PMH_ORDER_COST_M
#define PMH_ORDER_COST_M 7.0   // ProbMinHash set cost ~ n + c m (coupon phase) for the LPT order
#endif

using namespace pmh;

namespace {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return set_error(PMH_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define PMH_CUDA(call)                                  \
  do {                                                  \
    cudaError_t _e = (call);                            \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)
// for functions returning cudaError_t
#define PMH_CUDA_E(call)                 \
  do {                                   \
    cudaError_t _e = (call);             \
    if (_e != cudaSuccess) return _e;    \
  } while (0)


// ---- constant tables (glibc on the host, uploaded once per device and m) --
struct DevTables {
  Tables t{};
  void* mem = nullptr;
};

std::mutex g_mu;
std::map<std::tuple<int, int, int64_t>, DevTables> g_tables;

void trunc_consts(double lam, TruncExpConsts* c) {  // K:186-191
  c->lam = lam;
  c->c1 = std::expm1(lam) / lam;
  c->c2 = std::log(2.0 / (1.0 + std::exp(-lam))) / lam;
  c->c3 = -std::expm1(-lam) / lam;
}

int get_tables(int family, int64_t m, const Tables** out) {
  int dev = 0;
  PMH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_tuple(dev, family, m);
  auto it = g_tables.find(key);
  if (it != g_tables.end()) { *out = &it->second.t; return PMH_OK; }
  DevTables dt;
  if (family == FAM_PMH3 && m >= 2) {
    trunc_consts(std::log1p(1.0 / ((double)m - 1.0)), &dt.t.c3);  // K:458-459
  } else if (family == FAM_PMH2) {
    std::vector<double> beta(m + 1, 0.0);
    for (int64_t i = 2; i <= m; i++) beta[i] = (double)m / ((double)(m - i) + 1.0);  // K:418-420
    PMH_CUDA(cudaMalloc(&dt.mem, sizeof(double) * (m + 1)));
    PMH_CUDA(cudaMemcpy(dt.mem, beta.data(), sizeof(double) * (m + 1), cudaMemcpyHostToDevice));
    dt.t.beta = (const double*)dt.mem;
  } else if (family == FAM_PMH4 && m >= 2) {  // K:568-579
    std::vector<TruncExpConsts> c4(m);
    std::vector<double> gam(m, 0.0), dgam(m, 0.0);
    const double lam1 = std::log1p(1.0 / ((double)m - 1.0));
    for (int64_t i = 1; i < m; i++) {
      trunc_consts(std::log1p(1.0 / (double)(m - i)), &c4[i]);
      gam[i] = std::log1p((double)i / (double)(m - i)) / lam1;
    }
    for (int64_t i = 1; i < m; i++) dgam[i] = gam[i] - gam[i - 1];
    c4[0] = c4[m > 1 ? 1 : 0];
    dt.t.delta = 1.0 / lam1;
    const size_t bc = sizeof(TruncExpConsts) * m, bg = sizeof(double) * m;
    PMH_CUDA(cudaMalloc(&dt.mem, bc + 2 * bg));
    char* p = (char*)dt.mem;
    PMH_CUDA(cudaMemcpy(p, c4.data(), bc, cudaMemcpyHostToDevice));
    PMH_CUDA(cudaMemcpy(p + bc, gam.data(), bg, cudaMemcpyHostToDevice));
    PMH_CUDA(cudaMemcpy(p + bc + bg, dgam.data(), bg, cudaMemcpyHostToDevice));
    dt.t.c4 = (const TruncExpConsts*)p;
    dt.t.gam = (const double*)(p + bc);
    dt.t.dgam = (const double*)(p + bc + bg);
  }
  // the uploads above are synchronous copies from pageable memory, which may
  // return before the DMA lands; the kernels that read the tables run on
  // non-blocking streams that nothing orders after it, so wait here (once per
  // device, family and m) before publishing the table
  if (dt.mem) PMH_CUDA(cudaDeviceSynchronize());
  auto res = g_tables.emplace(key, dt);
  *out = &res.first->second.t;
  return PMH_OK;
}

// Test hook: PMH_TEST_REJECT_CAP / PMH_TEST_COUPON_CAP lower the device loop
// caps (pmh_device.cuh) so a test can drive RandomnessFailureError; read once
// per device.  Unset (always, outside tests) the reference caps apply.
std::map<int, bool> g_caps_applied;
int apply_test_caps() {
  int dev = 0;
  PMH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_caps_applied[dev]) return PMH_OK;
  if (const char* ev = getenv("PMH_TEST_REJECT_CAP")) {
    const int v = atoi(ev);
    PMH_CUDA(cudaMemcpyToSymbol(g_reject_cap, &v, sizeof(v)));
  }
  if (const char* ev = getenv("PMH_TEST_COUPON_CAP")) {
    const long long v = atoll(ev);
    PMH_CUDA(cudaMemcpyToSymbol(g_coupon_cap_override, &v, sizeof(v)));
  }
  g_caps_applied[dev] = true;
  return PMH_OK;
}

int family_of(int algo) {
  switch (algo) {
    case ALG_PMH1: case ALG_PMH1A: case ALG_UW1: case ALG_UW1A: return FAM_PMH1;
    case ALG_PMH2: case ALG_UW2: return FAM_PMH2;
    case ALG_PMH3: case ALG_PMH3A: return FAM_PMH3;
    case ALG_PMH4: return FAM_PMH4;
    case ALG_UW3: case ALG_UW3A: return FAM_UW3;
    case ALG_UW4: return FAM_UW4;
    default: return 0;
  }
}

bool is_unweighted(int algo) { return algo >= ALG_MINHASH; }
bool reports_buffer(int algo) {
  return algo == ALG_PMH1A || algo == ALG_PMH3A || algo == ALG_UW1A || algo == ALG_UW3A;
}
int64_t min_m(int algo) {
  switch (algo) {
    case ALG_PMH3: case ALG_PMH3A: case ALG_PMH4: case ALG_UW3: case ALG_UW3A:
    case ALG_UW4: case ALG_SUPERMINHASH: return 2;
    default: return 1;
  }
}

template <int F>
cudaError_t launch_family(const SketchArgs& a0, cudaStream_t st) {
  const int64_t grid0 = a0.nsets < 2147483647LL ? a0.nsets : 2147483647LL;
  if constexpr (family_uses_fy(F)) {
    // large m: 16 warps per set on 16-bit Fisher-Yates maps, or (beyond what
    // that layout holds) 8 warps on 16-bit maps
    if (sketch_use_big(F, a0.m) || sketch_fy16_256(F, a0.m)) {
      const bool big = sketch_use_big(F, a0.m);
      const int nt = big ? SKETCH_THREADS_BIG : SKETCH_THREADS;
      const size_t smem = sketch_smem_bytes(F, a0.m, nt, true);
      if (smem > SMEM_DYN_MAX) return cudaErrorInvalidValue;
      auto kern = big ? sketch_sets_kernel<F, SKETCH_THREADS_BIG, true>
                      : sketch_sets_kernel<F, SKETCH_THREADS, true>;
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
      if (e != cudaSuccess) return e;
      kern<<<(unsigned)grid0, nt, smem, st>>>(a0);
      return cudaGetLastError();
    }
  }
  const SketchArgs& a = a0;
  const int threads = SKETCH_THREADS;
  const size_t smem = sketch_smem_bytes(F, a.m, threads);
  if (smem > SMEM_DYN_MAX) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(sketch_sets_kernel<F>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = a.nsets < 2147483647LL ? a.nsets : 2147483647LL;
  sketch_sets_kernel<F><<<(unsigned)grid, threads, smem, st>>>(a);
  return cudaGetLastError();
}

template <int C, bool EXPO>
cudaError_t launch_pmin_c(const PMinArgs& a, cudaStream_t st) {
  const size_t smem = sizeof(Slot) * (size_t)a.m;
  cudaError_t e = cudaFuncSetAttribute(pminhash_kernel<C, EXPO>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t grid = a.nsets < 2147483647LL ? a.nsets : 2147483647LL;
  pminhash_kernel<C, EXPO><<<(unsigned)grid, PMIN_THREADS, smem, st>>>(a);
  return cudaGetLastError();
}

template <bool EXPO>
cudaError_t launch_pminhash(const PMinArgs& a, cudaStream_t st) {
  if (a.m % PM64_C == 0 && a.m / PM64_C <= PMIN_THREADS) {
    const size_t smem = sizeof(Slot) * (size_t)a.m + sizeof(uint2) * PM64_CQ * (PMIN_THREADS / 32);
    cudaError_t e = cudaFuncSetAttribute(pminhash64_kernel<EXPO>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int64_t grid = a.nsets < 2147483647LL ? a.nsets : 2147483647LL;
    pminhash64_kernel<EXPO><<<(unsigned)grid, PMIN_THREADS, smem, st>>>(a);
    return cudaGetLastError();
  }
  // C = components per thread: 32 for m >= 1024 (one warp per group at
  // m = 1024, 8 groups per CTA), else the power of two giving ~32 threads per
  // group; m <= 256 * 32 required
  int64_t c = 1;
  while (a.m > 32 * c && c < 32) c *= 2;
  if (a.m > (int64_t)PMIN_THREADS * c) return cudaErrorInvalidValue;
  switch (c) {
    case 1: return launch_pmin_c<1, EXPO>(a, st);
    case 2: return launch_pmin_c<2, EXPO>(a, st);
    case 4: return launch_pmin_c<4, EXPO>(a, st);
    case 8: return launch_pmin_c<8, EXPO>(a, st);
    case 16: return launch_pmin_c<16, EXPO>(a, st);
    default: return launch_pmin_c<32, EXPO>(a, st);
  }
}

// Build the LPT set order on `st` into workspace: int32 order[nsets], 64 u32
// bucket cursors, u32 counts[2] ([0] = number of sets with n > small_n, which
// form the order prefix).  small_n < 0 disables the small-set split.
struct OrderWs {
  int32_t* order = nullptr;
  unsigned* counts = nullptr;          // [0] #sets n > small_n, [1] #sets n >= big_n
  unsigned long long* ctr = nullptr;   // two work counters
  void* mem = nullptr;
};

cudaError_t build_order(const int64_t* offsets, int64_t nsets, int64_t c, int64_t small_n,
                        int64_t big_n, cudaStream_t st, OrderWs* ow) {
  void* ws = nullptr;
  const size_t hb = sizeof(unsigned) * (ORDER_BUCKETS + 4) + sizeof(unsigned long long) * 2;
  cudaError_t e = cudaMallocAsync(&ws, hb + sizeof(int32_t) * (size_t)nsets, st);
  if (e != cudaSuccess) return e;
  unsigned* hist = (unsigned*)ws;
  unsigned* counts = hist + ORDER_BUCKETS;
  unsigned long long* ctr = (unsigned long long*)(hist + ORDER_BUCKETS + 4);
  int32_t* order = (int32_t*)((char*)ws + hb);
  if ((e = cudaMemsetAsync(hist, 0, hb, st)) != cudaSuccess) return e;
  int64_t blocks = (nsets + 255) / 256;
  if (blocks > 1184) blocks = 1184;
  order_hist_kernel<<<(unsigned)blocks, 256, 0, st>>>(offsets, nsets, c, small_n, big_n, hist,
                                                      counts);
  order_scan_kernel<<<1, 32, 0, st>>>(hist);
  order_scatter_kernel<<<(unsigned)blocks, 256, 0, st>>>(offsets, nsets, c, small_n, hist, order);
  ow->order = order;
  ow->counts = counts;
  ow->ctr = ctr;
  ow->mem = ws;
  return cudaGetLastError();
}

// Keep the stream-ordered allocator's memory resident between calls (the
// default release threshold 0 would unmap the workspace at every sync).
std::map<int, bool> g_pool_set;
void ensure_pool_retained() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_pool_set[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  g_pool_set[dev] = true;
}

// A fork event private to one call: the shared per-device streams below may be
// used by several host threads at once (ctypes releases the GIL), so the
// event that orders a shared stream after the CALLER's stream must not be
// shared -- another thread's record could land between this call's record and
// its wait.  (Join events are recorded on the shared stream itself, where a
// later record only waits for more of the same stream: still correct.)
// Destroying it right after the wait is legal; the wait keeps its snapshot.
struct ForkEvent {
  cudaEvent_t e = nullptr;
  ForkEvent() { cudaEventCreateWithFlags(&e, cudaEventDisableTiming); }
  ~ForkEvent() { if (e) cudaEventDestroy(e); }
  ForkEvent(const ForkEvent&) = delete;
  ForkEvent& operator=(const ForkEvent&) = delete;
};

// per-device auxiliary stream + events for the concurrent small-set kernel
struct AuxStream {
  cudaStream_t s = nullptr;
  cudaEvent_t join = nullptr;
};
// keyed by (device, slot): slot 0 serves caller streams, slot k + 1 the k-th
// internal lane of pmh_sketch_csr_multi_async (so concurrent variants do not
// serialise their small-set kernels through one stream)
std::map<std::pair<int, int>, AuxStream> g_aux;

int get_aux(AuxStream** out, int slot = 0) {
  int dev = 0;
  PMH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_aux.find({dev, slot});
  if (it == g_aux.end()) {
    AuxStream a;
    // highest priority: the small-set kernel's (few, latency-bound) CTAs are
    // placed before the pending CTAs of the big kernel, so they run beside it
    // from the start instead of as a tail
    int least = 0, greatest = 0;
    PMH_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    PMH_CUDA(cudaStreamCreateWithPriority(&a.s, cudaStreamNonBlocking, greatest));
    PMH_CUDA(cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming));
    it = g_aux.emplace(std::make_pair(dev, slot), a).first;
  }
  *out = &it->second;
  return PMH_OK;
}

// Split workspace for the largest sets (pmh_split.cuh): slot table, part
// prefix and counters, from the stream-ordered pool.
struct SplitWs {
  SplitArgs sp{};
  char* mem = nullptr;
};
cudaError_t split_setup(const int64_t* offsets, const int32_t* order, int64_t nsets, int64_t c_off,
                        int64_t split_n, int64_t split_cap, int64_t m, int64_t* stats,
                        long long cta_slots, cudaStream_t st, SplitWs* ws) {
  const size_t bt = sizeof(Slot) * (size_t)split_cap * (size_t)m;
  const size_t bp = sizeof(int64_t) * (size_t)(split_cap + 1);
  cudaError_t e = cudaMallocAsync((void**)&ws->mem, bt + bp + 4 * sizeof(long long), st);
  if (e != cudaSuccess) return e;
  SplitArgs& sp = ws->sp;
  sp.offsets = offsets;
  sp.order = order;
  sp.nsets = nsets;
  sp.c_off = c_off;
  sp.split_n = split_n;
  sp.split_cap = split_cap;
  sp.m = m;
  sp.gtab = reinterpret_cast<Slot*>(ws->mem);
  sp.part_base = reinterpret_cast<int64_t*>(ws->mem + bt);
  sp.info = reinterpret_cast<long long*>(ws->mem + bt + bp);
  sp.stats = stats;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  split_prep_kernel<<<1, 1024, 0, st>>>(sp, cta_slots);
  split_init_kernel<<<(unsigned)(sms * 4), 256, 0, st>>>(sp);
  return cudaGetLastError();
}

// P-MinHash with its largest sets split across CTAs: prep and table init on
// `st`, then the split kernel on `st` beside the regular kernel (remaining
// sets) on the auxiliary stream, then the ids of the split sets.
template <bool EXPO>
cudaError_t launch_pminhash_split(PMinArgs a, int64_t split_n, int64_t split_cap,
                                  cudaStream_t st, int aux_slot) {
  AuxStream* aux = nullptr;
  if (get_aux(&aux, aux_slot) != PMH_OK) return cudaErrorUnknown;
  const size_t smem = sizeof(Slot) * (size_t)a.m + sizeof(uint2) * PM64_CQ * (PMIN_THREADS / 32);
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(pminhash64_split_kernel<EXPO>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
    return e;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pminhash64_split_kernel<EXPO>,
                                                PMIN_THREADS, smem);
  if (per_sm < 1) per_sm = 1;
  SplitWs ws;
  if ((e = split_setup(a.offsets, a.order, a.nsets, 0, split_n, split_cap, a.m, a.stats,
                       (long long)sms * per_sm, st, &ws)) != cudaSuccess)
    return e;
  a.split_info = ws.sp.info;
  {
    ForkEvent fork;
    PMH_CUDA_E(cudaEventRecord(fork.e, st));
    PMH_CUDA_E(cudaStreamWaitEvent(aux->s, fork.e, 0));
  }
  if ((e = launch_pminhash<EXPO>(a, aux->s)) != cudaSuccess) return e;   // remaining sets
  pminhash64_split_kernel<EXPO><<<(unsigned)(sms * per_sm), PMIN_THREADS, smem, st>>>(a, ws.sp);
  split_finalize_kernel<<<(unsigned)(sms * 4), 256, 0, st>>>(ws.sp, a.ids, a.sig);
  PMH_CUDA_E(cudaEventRecord(aux->join, aux->s));
  PMH_CUDA_E(cudaStreamWaitEvent(st, aux->join, 0));
  cudaFreeAsync(ws.mem, st);
  return cudaGetLastError();
}

// per-device pool of internal streams for the concurrent multi-variant entry
struct LanePool {
  std::vector<cudaStream_t> s;
  std::vector<cudaEvent_t> done;
};
std::map<int, LanePool> g_lanes;

int get_lanes(int n, LanePool** out) {
  int dev = 0;
  PMH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  LanePool& p = g_lanes[dev];
  while ((int)p.s.size() < n) {
    cudaStream_t st;
    cudaEvent_t ev;
    PMH_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    PMH_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    p.s.push_back(st);
    p.done.push_back(ev);
  }
  *out = &p;
  return PMH_OK;
}

template <int F>
cudaError_t launch_small(const SketchArgs& a, cudaStream_t st) {
  if (wps_eligible(F, a.m)) {   // small m: the lean warp-per-set kernel (pmh_wps.cuh)
    const size_t smem = sizeof(WpsWarp) * (WPS_THREADS / 32);
    cudaError_t e = cudaFuncSetAttribute(sketch_wps_kernel<F>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int64_t grid = (a.nsets + (WPS_THREADS / 32) - 1) / (WPS_THREADS / 32);
    if (grid > 148 * 32) grid = 148 * 32;
    sketch_wps_kernel<F><<<(unsigned)grid, WPS_THREADS, smem, st>>>(a);
    return cudaGetLastError();
  }
  const size_t per_warp = small_warp_bytes(F, a.m);
  int wpc = (int)((96 * 1024) / per_warp);
  wpc = wpc < 1 ? 1 : (wpc > 4 ? 4 : wpc);
  const size_t smem = per_warp * (size_t)wpc;
  if (smem > SMEM_DYN_MAX) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(sketch_small_kernel<F>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int64_t grid = (a.nsets + wpc - 1) / wpc;
  if (grid > 148 * 16) grid = 148 * 16;
  sketch_small_kernel<F><<<(unsigned)grid, 32 * wpc, smem, st>>>(a);
  return cudaGetLastError();
}

// argument validation with the reference's error domain (sketch.py:96-114);
// runs before any CUDA call
bool is_baseline(int algo) { return algo == ALG_SUPERMINHASH || algo == ALG_OPH; }

int validate_sketch(int algo, int64_t m, const double* weights, int64_t nsets) {
  const int fam = family_of(algo);
  if (algo != ALG_PMINHASH && algo != ALG_MINHASH && !is_baseline(algo) && fam == 0)
    return set_error(PMH_ERR_INVALID, "unsupported algorithm id " + std::to_string(algo));
  if (m < min_m(algo))
    return set_error(PMH_ERR_INVALID, "signature size must be >= " + std::to_string(min_m(algo)));
  if (fam != 0 && (sketch_smem_bytes(fam, m, SKETCH_THREADS, sketch_fy16_256(fam, m)) > SMEM_DYN_MAX ||
                   (sketch_fy16_256(fam, m) && m >= 8192)))
    return set_error(PMH_ERR_INVALID, "signature size too large for the shared-memory slot table");
  // the P-MinHash launchers: the static kernel takes m % 64 == 0 up to
  // 64 * PMIN_THREADS, the generic one m <= 32 * PMIN_THREADS
  if ((algo == ALG_PMINHASH || algo == ALG_MINHASH) &&
      !(m <= 32LL * PMIN_THREADS || (m % PM64_C == 0 && m <= 64LL * PMIN_THREADS)))
    return set_error(PMH_ERR_INVALID, "signature size too large for the P-MinHash kernel");
  if (algo == ALG_OPH && sizeof(Slot) * (size_t)m > SMEM_DYN_MAX)
    return set_error(PMH_ERR_INVALID, "signature size too large for the OPH kernel");
  if (m > 65535) return set_error(PMH_ERR_INVALID, "signature size must be <= 65535");
  if (nsets < 0) return set_error(PMH_ERR_INVALID, "negative set count");
  if (nsets > 0 && !is_unweighted(algo) && !weights)
    return set_error(PMH_ERR_INVALID, "weighted algorithm requires weights");
  return PMH_OK;
}

}  // namespace

extern "C" {

int pmh_version(void) { return 100; }

const char* pmh_last_error(void) { return g_last_error.c_str(); }

int pmh_status_reset(int64_t* d_status, void* stream) {
  const long long init[2] = {0, 0x7FFFFFFFFFFFFFFFLL};
  // small pageable copy: the driver stages it, stream-ordered
  PMH_CUDA(cudaMemcpyAsync(d_status, init, sizeof(init), cudaMemcpyHostToDevice,
                           (cudaStream_t)stream));
  return PMH_OK;
}

int pmh_status_check(const int64_t* d_status, int64_t* err_set, void* stream) {
  long long h[2] = {0, 0};
  PMH_CUDA(cudaMemcpyAsync(h, d_status, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  PMH_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (err_set) *err_set = -1;
  if (h[1] != 0x7FFFFFFFFFFFFFFFLL) {
    if (err_set) *err_set = h[1];
    if (h[0] & ERRF_RANDOMNESS)
      return set_error(PMH_ERR_RANDOMNESS, "rejection or coupon loop exceeded its cap in set " +
                                               std::to_string(h[1]));
    return set_error(PMH_ERR_EMPTY, "cannot sketch an empty set (set " + std::to_string(h[1]) + ")");
  }
  return PMH_OK;
}

static int sketch_async_impl(int algo, int64_t m, const uint64_t* ids, const double* weights,
                             const int64_t* offsets, int64_t nsets, uint64_t* sig_out,
                             int64_t* stats_out, int64_t* d_status, cudaStream_t st,
                             int aux_slot, const double* setw);

// per-set total weights into a stream-ordered pool buffer (nullptr on error)
static double* set_weights_tmp(const double* weights, const int64_t* offsets, int64_t nsets,
                               cudaStream_t st) {
  ensure_pool_retained();
  double* d = nullptr;
  if (cudaMallocAsync((void**)&d, sizeof(double) * (size_t)nsets, st) != cudaSuccess) return nullptr;
  int64_t grid = nsets < 148 * 16 ? nsets : 148 * 16;
  set_weights_kernel<<<(unsigned)grid, 256, 0, st>>>(weights, offsets, nsets, d);
  if (cudaGetLastError() != cudaSuccess) { cudaFreeAsync(d, st); return nullptr; }
  return d;
}

static bool uses_set_weights(int algo) {
  return algo == ALG_PMINHASH || algo == ALG_PMH1 || algo == ALG_PMH1A || algo == ALG_PMH2 ||
         algo == ALG_PMH3 || algo == ALG_PMH3A || algo == ALG_PMH4;
}

int pmh_sketch_csr_async(int algo, int64_t m, const uint64_t* ids,
                         const double* weights, const int64_t* offsets,
                         int64_t nsets, uint64_t* sig_out, int64_t* stats_out,
                         int64_t* d_status, void* stream) {
  return sketch_async_impl(algo, m, ids, weights, offsets, nsets, sig_out, stats_out, d_status,
                           (cudaStream_t)stream, 0, nullptr);
}

int pmh_sketch_csr_w_async(int algo, int64_t m, const uint64_t* ids, const double* weights,
                           const int64_t* offsets, int64_t nsets, const double* set_weights,
                           uint64_t* sig_out, int64_t* stats_out, int64_t* d_status,
                           void* stream) {
  return sketch_async_impl(algo, m, ids, weights, offsets, nsets, sig_out, stats_out, d_status,
                           (cudaStream_t)stream, 0, set_weights);
}

int pmh_set_weights(const double* weights, const int64_t* offsets, int64_t nsets, double* out,
                    void* stream) {
  if (nsets < 0) return set_error(PMH_ERR_INVALID, "negative set count");
  if (nsets == 0) return PMH_OK;
  if (!weights || !offsets || !out) return set_error(PMH_ERR_INVALID, "weights, offsets, out required");
  int64_t grid = nsets < 148 * 16 ? nsets : 148 * 16;
  set_weights_kernel<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(weights, offsets, nsets, out);
  PMH_CUDA(cudaGetLastError());
  return PMH_OK;
}

int pmh_sketch_csr_multi_async(const int* algos, int nalgos, int64_t m, const uint64_t* ids,
                               const double* weights, const int64_t* offsets, int64_t nsets,
                               uint64_t* const* sig_outs, int64_t* const* stats_outs,
                               int64_t* d_status, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (nalgos < 1 || nalgos > 32 || !algos || !sig_outs)
    return set_error(PMH_ERR_INVALID, "1..32 algorithms with outputs required");
  ensure_pool_retained();
  for (int k = 0; k < nalgos; k++) {
    int vrc = validate_sketch(algos[k], m, weights, nsets);
    if (vrc != PMH_OK) return vrc;
  }
  if (nsets == 0) return PMH_OK;
  if (!d_status) return set_error(PMH_ERR_INVALID, "status buffer required");
  LanePool* lp = nullptr;
  int rc = get_lanes(nalgos, &lp);
  if (rc) return rc;
  // the per-set total weights once for every variant (each kernel would
  // otherwise re-read all weights for its threshold guess)
  int n_w = 0;
  for (int k = 0; k < nalgos; k++) n_w += uses_set_weights(algos[k]);
  double* setw = nullptr;
  if (weights && n_w > 1) {
    setw = set_weights_tmp(weights, offsets, nsets, st);
    if (!setw) return set_error(PMH_ERR_CUDA, "set weights");
  }
  ForkEvent fork;
  PMH_CUDA(cudaEventRecord(fork.e, st));
  // the P-MinHash-type variants (one long, tail-light kernel) last: their
  // CTAs fill the tails of the ProbMinHash kernels launched before them
  std::vector<int> order;
  for (int pass = 0; pass < 2; pass++)
    for (int k = 0; k < nalgos; k++) {
      const bool pmin = algos[k] == ALG_PMINHASH || algos[k] == ALG_MINHASH;
      if (pmin == (pass == 1)) order.push_back(k);
    }
  for (int k : order) {
    PMH_CUDA(cudaStreamWaitEvent(lp->s[k], fork.e, 0));
    rc = sketch_async_impl(algos[k], m, ids, weights, offsets, nsets, sig_outs[k],
                           stats_outs ? stats_outs[k] : nullptr, d_status, lp->s[k], k + 1,
                           uses_set_weights(algos[k]) ? setw : nullptr);
    PMH_CUDA(cudaEventRecord(lp->done[k], lp->s[k]));
    PMH_CUDA(cudaStreamWaitEvent(st, lp->done[k], 0));
    if (rc != PMH_OK) { if (setw) cudaFreeAsync(setw, st); return rc; }
  }
  if (setw) cudaFreeAsync(setw, st);   // after the join: every variant is done with it
  return PMH_OK;
}

static int sketch_async_impl(int algo, int64_t m, const uint64_t* ids, const double* weights,
                             const int64_t* offsets, int64_t nsets, uint64_t* sig_out,
                             int64_t* stats_out, int64_t* d_status, cudaStream_t st,
                             int aux_slot, const double* setw) {
  // the stream-ordered workspaces of the call (set order, split tables) must
  // stay mapped between calls: with the pool's default release threshold 0
  // they are unmapped at every synchronisation and re-mapped by the next
  // call, a host-side stall of up to ~40 ms before its first kernel
  ensure_pool_retained();
  const int fam = family_of(algo);
  int vrc = validate_sketch(algo, m, weights, nsets);
  if (vrc != PMH_OK) return vrc;
  if (nsets == 0) return PMH_OK;
  if (!d_status) return set_error(PMH_ERR_INVALID, "status buffer required");
  unsigned long long* flags = reinterpret_cast<unsigned long long*>(d_status);
  long long* d_err_set = reinterpret_cast<long long*>(d_status + 1);
  {
    const int crc = apply_test_caps();
    if (crc != PMH_OK) return crc;
  }

  cudaError_t e;
  if (is_baseline(algo)) {
    BaseArgs b{ids, offsets, nsets, m, sig_out, stats_out, d_err_set, flags};
    const int64_t grid = nsets < 2147483647LL ? nsets : 2147483647LL;
    if (algo == ALG_OPH) {
      const size_t smem = sizeof(Slot) * (size_t)m;
      PMH_CUDA(cudaFuncSetAttribute(oph_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem));
      oph_kernel<<<(unsigned)grid, 256, smem, st>>>(b);
    } else {
      int threads = 256;
      size_t smem = sizeof(Slot) * (size_t)m + sizeof(int32_t) * (size_t)m * (threads / 32);
      while (smem > 200 * 1024 && threads > 32) {
        threads /= 2;
        smem = sizeof(Slot) * (size_t)m + sizeof(int32_t) * (size_t)m * (threads / 32);
      }
      if (smem > SMEM_DYN_MAX) return set_error(PMH_ERR_INVALID, "signature size too large");
      PMH_CUDA(cudaFuncSetAttribute(superminhash_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      superminhash_kernel<<<(unsigned)grid, threads, smem, st>>>(b);
    }
    PMH_CUDA(cudaGetLastError());
    return PMH_OK;
  }
  const bool pmin = algo == ALG_PMINHASH || algo == ALG_MINHASH;
  // P-MinHash splits its largest sets across CTAs (static kernel only): sets
  // with n >= split_n (a power of two, so with cost offset 0 they form a
  // prefix of the LPT order), at most split_cap of them.  Parts of 4096
  // elements: one part is ~2 ms of one CTA at m = 1024, so a small batch (a
  // rank's shard, ~1,200 sets) is not left waiting on a few long parts
  // (1/8 of configs[1]: 11.6 -> 11.0 ms; the whole batch unchanged, 71.4 ms)
  const bool pm_static = pmin && m % PM64_C == 0 && m / PM64_C <= PMIN_THREADS;
  int64_t split_n = 4096, split_cap = 1024;
  if (const char* ev = getenv("PMH_PM64_SPLIT_N")) split_n = atoll(ev);
  if (const char* ev = getenv("PMH_PM64_SPLIT_CAP")) split_cap = atoll(ev);
  if (split_cap > (1LL << 24) / m) split_cap = (1LL << 24) / m;
  const bool pm_split = pm_static && split_n >= 64 && (split_n & (split_n - 1)) == 0 &&
                        split_cap > 0;
  OrderWs ow;
#ifndef PMH_FLAT
#define PMH_FLAT 1
#endif
  // ProbMinHash3 / unweighted 3 at power-of-two m: the flat point-parallel
  // kernel takes the sets up to PMH_FLAT_NMAX elements (instead of the
  // warp-per-set kernels), concurrently with the CTA kernel on the larger ones
  // For the UNWEIGHTED family the lane-per-element CTA path is faster from 256
  // equal-weight elements on (configs[2], m = 4096, n = 1000: 63.8 -> 34.3 ms;
  // 1.5-2x at every m), and at m > 256 its warp-cooperative path also beats
  // the flat kernel on smaller sets (tools/uw_sweep.py): flat only at
  // m <= 256, for sets below 256 elements.
  const bool flat = PMH_FLAT && !pmin && flat_eligible(fam, m) && !(fam == FAM_UW3 && m > 256);
  const int64_t flat_nmax = fam == FAM_UW3 ? 255 : (int64_t)PMH_FLAT_NMAX;
  // cost offset: ProbMinHash families pay ~m ln m points per set regardless of n
  e = build_order(offsets, nsets, pmin ? 0 : (int64_t)(PMH_ORDER_COST_M * (double)m),
                  pmin ? -1 : (flat ? flat_nmax : small_n_for(fam, m)),
                  pm_split ? split_n : 4096, st, &ow);
  if (e != cudaSuccess) return cuda_fail(e, "set ordering");
  int32_t* order = ow.order;
  void* order_ws = ow.mem;
  if (pmin) {
    PMinArgs a{ids, algo == ALG_PMINHASH ? weights : nullptr, offsets, order, nsets, m,
               sig_out, stats_out, d_err_set};
    a.setw = algo == ALG_PMINHASH ? setw : nullptr;
    if (!pm_split) {
      e = algo == ALG_PMINHASH ? launch_pminhash<true>(a, st) : launch_pminhash<false>(a, st);
    } else {
      e = algo == ALG_PMINHASH
              ? launch_pminhash_split<true>(a, split_n, split_cap, st, aux_slot)
              : launch_pminhash_split<false>(a, split_n, split_cap, st, aux_slot);
    }
  } else {
    const Tables* tp = nullptr;
    int rc = get_tables(fam, m, &tp);
    if (rc) { cudaFreeAsync(order_ws, st); return rc; }
    SketchArgs a{};
    a.ids = ids;
    a.w = is_unweighted(algo) ? nullptr : weights;
    a.offsets = offsets;
    a.order = order;
    a.nsets = nsets;
    a.m = m;
    a.sig = sig_out;
    a.stats = stats_out;
    a.err_flags = flags;
    a.err_set = d_err_set;
    a.T = *tp;
    a.setw = is_unweighted(algo) ? nullptr : setw;
    // threshold guess m (ln m + c) / W, measured on config 2 (c = 2/3/4/5):
    // c = 3 best for ProbMinHash 1/2/4 (2-6 % faster PMH2/PMH4 than c = 4;
    // ~5% of sets retry with 4 tg), c = 4 for ProbMinHash 3 (-3% vs 3)
    a.tconst = fam == FAM_PMH3 ? 4.0 : 3.0;
    if (const char* ev = getenv("PMH_TCONST")) a.tconst = atof(ev);   // tuning hook
    a.counts = ow.counts;
    // small sets run warp-per-set on the auxiliary stream, concurrently with
    // the CTA-per-set kernel on `st` (fork/join with events)
    AuxStream* aux = nullptr;
    rc = get_aux(&aux, aux_slot);
    if (rc) { cudaFreeAsync(order_ws, st); return rc; }
    {
      ForkEvent fork;
      PMH_CUDA(cudaEventRecord(fork.e, st));
      PMH_CUDA(cudaStreamWaitEvent(aux->s, fork.e, 0));
    }
    auto big = [&]() {
      switch (fam) {
        case FAM_PMH1: return launch_family<FAM_PMH1>(a, st);
        case FAM_PMH2: return launch_family<FAM_PMH2>(a, st);
        case FAM_PMH3: return launch_family<FAM_PMH3>(a, st);
        case FAM_PMH4: return launch_family<FAM_PMH4>(a, st);
        case FAM_UW3: return launch_family<FAM_UW3>(a, st);
        default: return launch_family<FAM_UW4>(a, st);
      }
    };
    auto small = [&]() {
      switch (fam) {
        case FAM_PMH1: return launch_small<FAM_PMH1>(a, aux->s);
        case FAM_PMH2: return launch_small<FAM_PMH2>(a, aux->s);
        case FAM_PMH3: return launch_small<FAM_PMH3>(a, aux->s);
        case FAM_PMH4: return launch_small<FAM_PMH4>(a, aux->s);
        case FAM_UW3: return launch_small<FAM_UW3>(a, aux->s);
        default: return launch_small<FAM_UW4>(a, aux->s);
      }
    };
    // the largest sets split across CTAs first (pmh_split.cuh): parts of
    // split_n elements (each part pays its own coupon phase, ~m ln m points,
    // so parts are larger than P-MinHash's)
    SplitWs sws;
    int64_t sp_n = 131072, sp_cap = 1024;
    if (const char* ev = getenv("PMH_SPLIT_N")) sp_n = atoll(ev);
    if (const char* ev = getenv("PMH_SPLIT_CAP")) sp_cap = atoll(ev);
    if (sp_cap > (1LL << 24) / m) sp_cap = (1LL << 24) / m;
    auto split = [&]() -> cudaError_t {
      const bool fy16 = sketch_fy16_256(fam, m);
      const size_t smem = sketch_smem_bytes(fam, m, SKETCH_THREADS, fy16);
      int dev = 0, sms = 148, per_sm = 1;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)smem);
        if (e2 != cudaSuccess) return e2;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SKETCH_THREADS, smem);
        if (per_sm < 1) per_sm = 1;
        e2 = split_setup(offsets, order, nsets, (int64_t)(PMH_ORDER_COST_M * (double)m), sp_n, sp_cap, m,
                         stats_out, (long long)sms * per_sm, st, &sws);
        if (e2 != cudaSuccess) return e2;
        a.split_info = sws.sp.info;
        kern<<<(unsigned)(sms * per_sm), SKETCH_THREADS, smem, st>>>(a, sws.sp);
        split_finalize_kernel<<<(unsigned)(sms * 4), 256, 0, st>>>(sws.sp, ids, sig_out);
        return cudaGetLastError();
      };
      switch (fam) {
        case FAM_PMH1: return go(sketch_split_kernel<FAM_PMH1>);
        case FAM_PMH2: return fy16 ? go(sketch_split_kernel<FAM_PMH2, true>)
                                   : go(sketch_split_kernel<FAM_PMH2>);
        case FAM_PMH3: return go(sketch_split_kernel<FAM_PMH3>);
        case FAM_PMH4: return fy16 ? go(sketch_split_kernel<FAM_PMH4, true>)
                                   : go(sketch_split_kernel<FAM_PMH4>);
        case FAM_UW3: return go(sketch_split_kernel<FAM_UW3>);
        default: return fy16 ? go(sketch_split_kernel<FAM_UW4, true>)
                             : go(sketch_split_kernel<FAM_UW4>);
      }
    };
    const bool do_split = sp_n >= 64 && sp_cap > 0;
    auto flat_launch = [&]() -> cudaError_t {   // the small partition, on the aux stream
      const size_t smem = sizeof(Slot) * (size_t)m;
      auto kern = fam == FAM_PMH3 ? sketch_flat_kernel<FAM_PMH3> : sketch_flat_kernel<FAM_UW3>;
      cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e2 != cudaSuccess) return e2;
      int64_t grid = nsets < 148 * 6 ? nsets : 148 * 6;
      kern<<<(unsigned)grid, FLAT_THREADS, smem, aux->s>>>(a);
      return cudaGetLastError();
    };
    // the small-set kernel first (see get_aux)
    e = flat ? flat_launch() : small();
    if (e == cudaSuccess && do_split) e = split();
    if (e == cudaSuccess) e = big();
    cudaEventRecord(aux->join, aux->s);
    cudaStreamWaitEvent(st, aux->join, 0);
    if (sws.mem) cudaFreeAsync(sws.mem, st);
  }
  cudaFreeAsync(order_ws, st);
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  if (stats_out && !reports_buffer(algo) && algo != ALG_PMINHASH && algo != ALG_MINHASH) {
    // the non-interleaved variants have no buffer (K:334-336): column 1 = 0
    PMH_CUDA(cudaMemset2DAsync(stats_out + 1, 3 * sizeof(int64_t), 0, sizeof(int64_t),
                               (size_t)nsets, st));
  }
  return PMH_OK;
}

int pmh_sketch_csr(int algo, int64_t m, const uint64_t* ids,
                   const double* weights, const int64_t* offsets,
                   int64_t nsets, uint64_t* sig_out, int64_t* stats_out,
                   int64_t* err_set, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (err_set) *err_set = -1;
  int vrc = validate_sketch(algo, m, weights, nsets);
  if (vrc != PMH_OK) return vrc;
  if (nsets == 0) return PMH_OK;
  ensure_pool_retained();
  int64_t* d_status = nullptr;
  PMH_CUDA(cudaMallocAsync((void**)&d_status, 16, st));
  int rc = pmh_status_reset(d_status, st);
  if (rc == PMH_OK)
    rc = pmh_sketch_csr_async(algo, m, ids, weights, offsets, nsets, sig_out, stats_out,
                              d_status, st);
  if (rc == PMH_OK) rc = pmh_status_check(d_status, err_set, st);
  cudaFreeAsync(d_status, st);
  return rc;
}

}  // extern "C"

namespace {
// per-device rotating pool of stream sets for the host entry points, so that
// consecutive asynchronous calls (pipelined batches) never share a stream
struct HostSet {
  cudaStream_t st = nullptr, cin = nullptr, cout = nullptr, cst[8] = {};
};
constexpr int HOST_SETS = 3;
std::map<int, std::vector<HostSet>> g_host_sets;
std::map<int, unsigned> g_host_next;
// per-device "kernels of the previous host call are done": a call's kernels
// wait on it (compute stays in call order, no interference between batches)
// while its copy-in does not (so it overlaps the previous batch's kernels)
std::map<int, cudaEvent_t> g_compute_done;

int get_compute_done(cudaEvent_t* out) {
  int dev = 0;
  PMH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEvent_t& ev = g_compute_done[dev];
  if (!ev) {
    PMH_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    PMH_CUDA(cudaEventRecord(ev, 0));
  }
  *out = ev;
  return PMH_OK;
}

int get_host_set(HostSet** out) {
  int dev = 0;
  PMH_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  std::vector<HostSet>& v = g_host_sets[dev];
  if (v.empty()) {
    v.resize(HOST_SETS);
    for (HostSet& h : v) {
      PMH_CUDA(cudaStreamCreateWithFlags(&h.st, cudaStreamNonBlocking));
      PMH_CUDA(cudaStreamCreateWithFlags(&h.cin, cudaStreamNonBlocking));
      PMH_CUDA(cudaStreamCreateWithFlags(&h.cout, cudaStreamNonBlocking));
      for (auto& c : h.cst) PMH_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
    }
  }
  *out = &v[g_host_next[dev]++ % HOST_SETS];
  return PMH_OK;
}
}  // namespace

extern "C" {

// Host-buffer entry (synchronous when ext_status == nullptr, else enqueue-only
// on `caller`, errors through ext_status).
static int host_multi_impl(const int* algos, int nalgos, int64_t m, const uint64_t* ids,
                           const double* weights, const int64_t* offsets, int64_t nsets,
                           int64_t nelems, uint64_t* const* sig_outs, int64_t* const* stats_outs,
                           int64_t* err_set, int64_t* ext_status, cudaStream_t caller) {
  if (err_set) *err_set = -1;
  if (nalgos < 1 || !algos || !sig_outs) return set_error(PMH_ERR_INVALID, "no algorithms");
  if (nsets < 0 || nelems < 0) return set_error(PMH_ERR_INVALID, "negative sizes");
  bool any_weighted = false;
  for (int k = 0; k < nalgos; k++) {
    int vrc = validate_sketch(algos[k], m, weights, nsets);
    if (vrc != PMH_OK) return vrc;
    any_weighted |= !is_unweighted(algos[k]);
  }
  if (nsets == 0) return PMH_OK;
  if (!ids || !offsets) return set_error(PMH_ERR_INVALID, "ids and offsets required");
  if (offsets[0] != 0) return set_error(PMH_ERR_INVALID, "offsets[0] must be 0");
  if (offsets[nsets] != nelems) return set_error(PMH_ERR_INVALID, "offsets[nsets] != nelems");
  for (int64_t s = 0; s < nsets; s++)  // host buffers: report empties up front
    if (offsets[s + 1] <= offsets[s]) {
      if (err_set) *err_set = s;
      return set_error(PMH_ERR_EMPTY, "cannot sketch an empty set (set " + std::to_string(s) + ")");
    }
  const bool weighted = any_weighted && weights;
  ensure_pool_retained();
  HostSet* hs = nullptr;
  {
    int prc = get_host_set(&hs);
    if (prc) return prc;
  }
  cudaStream_t st = hs->st, cin = hs->cin, cout = hs->cout;
  cudaEvent_t compute_done = nullptr;
  {
    int erc = get_compute_done(&compute_done);
    if (erc) return erc;
  }
  std::vector<cudaEvent_t> evs;
  auto mkev = [&]() {
    cudaEvent_t ev = nullptr;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    evs.push_back(ev);
    return ev;
  };
  // asynchronous calls do not wait for prior work on the caller's stream
  // (their inputs are host buffers): that is what lets batch i+1's copy-in
  // run under batch i's kernels; only their completion is joined back
  const size_t bi = sizeof(uint64_t) * (size_t)nelems, bw = weighted ? sizeof(double) * (size_t)nelems : 0,
               bo = sizeof(int64_t) * (size_t)(nsets + 1), bs = sizeof(uint64_t) * (size_t)nsets * (size_t)m,
               bst = sizeof(int64_t) * 3 * (size_t)nsets;
  const bool want_stats = stats_outs != nullptr;
  const size_t per_algo = bs + (want_stats ? bst : 0);
  char* d = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&d, bi + bw + bo + 16 + per_algo * (size_t)nalgos + 64, st);
  if (e != cudaSuccess) {
    for (auto ev : evs) cudaEventDestroy(ev);
    return cuda_fail(e, "cudaMallocAsync");
  }
  uint64_t* d_ids = (uint64_t*)d;
  double* d_w = (double*)(d + bi);
  int64_t* d_off = (int64_t*)(d + bi + bw);
  int64_t* d_status = ext_status ? ext_status : (int64_t*)(d + bi + bw + bo);
  char* d_out = d + bi + bw + bo + 16;
  int rc = PMH_OK;
  // Schedule (the copy-in is the long pole: 1.39 GB at ~55 GB/s for config 2):
  //  * offsets + status first, then the element arrays in NC set-chunks on
  //    the copy-in stream;
  //  * every ProbMinHash-type algorithm ("chunkable": its per-chunk kernels
  //    cost about the same as one whole-batch kernel) sketches each chunk as
  //    soon as it lands, on that chunk's stream, and the chunk's signature
  //    rows go back on the copy-out stream right away;
  //  * P-MinHash / MinHash (one long compute-bound kernel that chunking slows
  //    down) run over the whole batch once every chunk has landed, their
  //    D2H overlapping whatever still runs.
  e = cudaMemcpyAsync(d_off, offsets, bo, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) rc = cuda_fail(e, "H2D offsets");
  if (rc == PMH_OK && !ext_status) rc = pmh_status_reset(d_status, st);
  cudaEvent_t ev_meta = mkev();
  cudaEventRecord(ev_meta, st);
  cudaStreamWaitEvent(cin, ev_meta, 0);
  // synchronous calls chunk the copy-in so the batch's own kernels start
  // early; pipelined (async) calls copy in whole: their kernels wait for the
  // previous batch's anyway, and whole-batch kernels are cheaper than chunked
  int NC = (!ext_status && nsets >= 8 && nelems >= (1 << 20)) ? 4 : 1;
  if (const char* ev = getenv("PMH_H2D_CHUNKS")) {
    const int v = atoi(ev);
    if (v >= 1 && v <= 8 && nsets >= v) NC = v;
  }
  std::vector<int64_t> cut(NC + 1, 0);
  cut[NC] = nsets;
  for (int c = 1; c < NC; c++) {  // element-balanced set boundaries
    const int64_t target = nelems * c / NC;
    int64_t lo = cut[c - 1], hi = nsets;
    while (lo < hi) { const int64_t mid = (lo + hi) / 2; if (offsets[mid] < target) lo = mid + 1; else hi = mid; }
    cut[c] = lo;
  }
  auto chunkable = [&](int k) { return algos[k] != ALG_PMINHASH && algos[k] != ALG_MINHASH; };
  std::vector<cudaEvent_t> chunk_done;
  cudaStream_t* cst = hs->cst;
  for (int c = 0; c < NC && rc == PMH_OK; c++) {
    const int64_t e0 = offsets[cut[c]], e1 = offsets[cut[c + 1]];
    if (e1 > e0) {
      if ((e = cudaMemcpyAsync(d_ids + e0, ids + e0, sizeof(uint64_t) * (size_t)(e1 - e0),
                               cudaMemcpyHostToDevice, cin)) != cudaSuccess ||
          (weighted && (e = cudaMemcpyAsync(d_w + e0, weights + e0, sizeof(double) * (size_t)(e1 - e0),
                                            cudaMemcpyHostToDevice, cin)) != cudaSuccess)) {
        rc = cuda_fail(e, "H2D");
        break;
      }
    }
    cudaEvent_t ev = mkev();
    cudaEventRecord(ev, cin);
    cudaStreamWaitEvent(cst[c], ev, 0);
    cudaStreamWaitEvent(cst[c], compute_done, 0);
    const int64_t ns = cut[c + 1] - cut[c];
    // the chunk's per-set total weights once for its weighted variants
    int n_w = 0;
    for (int k = 0; k < nalgos; k++) n_w += chunkable(k) && uses_set_weights(algos[k]);
    double* setw = nullptr;
    if (weighted && n_w > 1 && ns > 0) {
      setw = set_weights_tmp(d_w, d_off + cut[c], ns, cst[c]);
      if (!setw) { rc = set_error(PMH_ERR_CUDA, "set weights"); break; }
    }
    for (int k = 0; k < nalgos && rc == PMH_OK && ns > 0; k++) {
      if (!chunkable(k)) continue;
      char* outk = d_out + per_algo * (size_t)k;
      uint64_t* sig0 = (uint64_t*)outk + (size_t)cut[c] * m;
      int64_t* st0 = want_stats ? (int64_t*)(outk + bs) + 3 * cut[c] : nullptr;
      rc = pmh_sketch_csr_w_async(algos[k], m, d_ids, weighted ? d_w : nullptr, d_off + cut[c], ns,
                                  uses_set_weights(algos[k]) ? setw : nullptr, sig0, st0, d_status,
                                  cst[c]);
      if (rc != PMH_OK) break;
      cudaEvent_t evk = mkev();
      cudaEventRecord(evk, cst[c]);
      cudaStreamWaitEvent(cout, evk, 0);
      const size_t rows = (size_t)ns * (size_t)m * sizeof(uint64_t);
      if ((e = cudaMemcpyAsync(sig_outs[k] + (size_t)cut[c] * m, sig0, rows, cudaMemcpyDeviceToHost,
                               cout)) != cudaSuccess ||
          (want_stats && stats_outs[k] &&
           (e = cudaMemcpyAsync(stats_outs[k] + 3 * cut[c], st0, sizeof(int64_t) * 3 * (size_t)ns,
                                cudaMemcpyDeviceToHost, cout)) != cudaSuccess)) {
        rc = cuda_fail(e, "D2H");
        break;
      }
    }
    if (setw) cudaFreeAsync(setw, cst[c]);
    cudaEvent_t evc = mkev();
    cudaEventRecord(evc, cst[c]);
    chunk_done.push_back(evc);
  }
  // whole-batch algorithms as soon as every chunk is resident (they overlap
  // the chunk streams' remaining work)
  cudaEvent_t ev_in = mkev();
  cudaEventRecord(ev_in, cin);
  cudaStreamWaitEvent(st, ev_in, 0);
  cudaStreamWaitEvent(st, compute_done, 0);
  for (int k = 0; k < nalgos && rc == PMH_OK; k++) {
    if (chunkable(k)) continue;
    char* outk = d_out + per_algo * (size_t)k;
    rc = pmh_sketch_csr_async(algos[k], m, d_ids, weighted ? d_w : nullptr, d_off, nsets,
                              (uint64_t*)outk, want_stats ? (int64_t*)(outk + bs) : nullptr,
                              d_status, st);
    if (rc != PMH_OK) break;
    cudaEvent_t ev = mkev();
    cudaEventRecord(ev, st);
    cudaStreamWaitEvent(cout, ev, 0);
    if ((e = cudaMemcpyAsync(sig_outs[k], outk, bs, cudaMemcpyDeviceToHost, cout)) != cudaSuccess ||
        (want_stats && stats_outs[k] &&
         (e = cudaMemcpyAsync(stats_outs[k], outk + bs, bst, cudaMemcpyDeviceToHost, cout)) != cudaSuccess)) {
      rc = cuda_fail(e, "D2H");
      break;
    }
  }
  for (cudaEvent_t evc : chunk_done) cudaStreamWaitEvent(st, evc, 0);
  cudaEventRecord(compute_done, st);   // this call's kernels, for the next call
  cudaEvent_t ev_end = mkev();
  cudaEventRecord(ev_end, cout);
  cudaStreamWaitEvent(st, ev_end, 0);
  if (ext_status) {
    cudaFreeAsync(d, st);
    cudaEvent_t join = mkev();
    cudaEventRecord(join, st);
    cudaStreamWaitEvent(caller, join, 0);
    for (auto ev : evs) cudaEventDestroy(ev);   // released once complete
    return rc;
  }
  if (rc == PMH_OK) rc = pmh_status_check(d_status, err_set, st);
  cudaFreeAsync(d, st);
  e = cudaStreamSynchronize(st);
  for (auto ev : evs) cudaEventDestroy(ev);
  if (rc == PMH_OK && e != cudaSuccess) rc = cuda_fail(e, "sync");
  return rc;
}

int pmh_sketch_csr_host_multi(const int* algos, int nalgos, int64_t m, const uint64_t* ids,
                              const double* weights, const int64_t* offsets, int64_t nsets,
                              int64_t nelems, uint64_t* const* sig_outs,
                              int64_t* const* stats_outs, int64_t* err_set) {
  return host_multi_impl(algos, nalgos, m, ids, weights, offsets, nsets, nelems, sig_outs,
                         stats_outs, err_set, nullptr, nullptr);
}

int pmh_sketch_csr_host_multi_async(const int* algos, int nalgos, int64_t m, const uint64_t* ids,
                                    const double* weights, const int64_t* offsets, int64_t nsets,
                                    int64_t nelems, uint64_t* const* sig_outs,
                                    int64_t* const* stats_outs, int64_t* d_status, void* stream) {
  if (!d_status) return set_error(PMH_ERR_INVALID, "status buffer required");
  return host_multi_impl(algos, nalgos, m, ids, weights, offsets, nsets, nelems, sig_outs,
                         stats_outs, nullptr, d_status, (cudaStream_t)stream);
}

int pmh_sketch_csr_host(int algo, int64_t m, const uint64_t* ids,
                        const double* weights, const int64_t* offsets,
                        int64_t nsets, int64_t nelems, uint64_t* sig_out,
                        int64_t* stats_out, int64_t* err_set) {
  uint64_t* const sigs[1] = {sig_out};
  int64_t* const stats[1] = {stats_out};
  return pmh_sketch_csr_host_multi(&algo, 1, m, ids, weights, offsets, nsets, nelems, sigs,
                                   stats_out ? stats : nullptr, err_set);
}

int pmh_count_equal(const uint64_t* a, const uint64_t* b, int64_t npairs,
                    int64_t m, int32_t* counts, void* stream) {
  if (m < 1 || npairs < 0) return set_error(PMH_ERR_INVALID, "bad sizes");
  if (npairs == 0) return PMH_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = 256;
  int64_t blocks = (npairs * 32 + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  count_equal_kernel<<<(unsigned)blocks, threads, 0, st>>>(a, b, npairs, m, counts);
  PMH_CUDA(cudaGetLastError());
  return PMH_OK;
}

int pmh_allpairs_tile(const uint64_t* sigs, int64_t n, int64_t m, int64_t r0,
                      int64_t r1, int64_t c0, int64_t c1, uint16_t* out,
                      int64_t ld, void* stream) {
  if (m < 1 || m > 65535 || r0 < 0 || r1 > n || c0 < 0 || c1 > n || r0 > r1 || c0 > c1)
    return set_error(PMH_ERR_INVALID, "bad tile bounds");
  if (r0 == r1 || c0 == c1) return PMH_OK;
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((unsigned)((c1 - c0 + AP_TILE - 1) / AP_TILE), (unsigned)((r1 - r0 + AP_TILE - 1) / AP_TILE));
  allpairs_tile_kernel<<<grid, 256, 0, st>>>(sigs, n, m, r0, r1, c0, c1, out, ld);
  PMH_CUDA(cudaGetLastError());
  return PMH_OK;
}

}  // extern "C"

namespace {
template <class Cmp>
int launch_allpairs_reduce(const uint64_t* rows, int64_t len, int64_t m, Cmp cmp, int64_t r0,
                           int64_t r1, int64_t c0, int64_t c1, int32_t thr, uint64_t* hist,
                           uint64_t* pairs, int64_t cap, uint64_t* cursor, cudaStream_t st,
                           const unsigned long long* gate = nullptr,
                           unsigned long long gate_cap = 0) {
  const size_t smem = 2 * sizeof(uint64_t) * AP_KS * (AP_TILE + 1) + sizeof(unsigned) * (size_t)(m + 1);
  PMH_CUDA(cudaFuncSetAttribute(allpairs_reduce_kernel<Cmp>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, allpairs_reduce_kernel<Cmp>, 256, smem);
  if (per_sm < 1) per_sm = 1;
  const int64_t ntiles = ((r1 - r0 + AP_TILE - 1) / AP_TILE) * ((c1 - c0 + AP_TILE - 1) / AP_TILE);
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > ntiles) grid = ntiles;
  allpairs_reduce_kernel<Cmp><<<(unsigned)grid, 256, smem, st>>>(
      rows, len, m, cmp, r0, r1, c0, c1, thr, (unsigned long long*)hist,
      (unsigned long long*)pairs, cap, (unsigned long long*)cursor, gate, gate_cap);
  PMH_CUDA(cudaGetLastError());
  return PMH_OK;
}

// Exact all-pairs counts in two stages (pmh_pminhash.cuh: allpairs_lo_kernel):
// low-32-bit compares over every pair, exact recount of the pairs with a
// low-word match, the exact single-stage reduction as a device-gated fallback
// when the candidate list overflows.  Stream-ordered, no host sync.
int launch_allpairs_exact2(const uint64_t* sigs, int64_t m, int64_t r0, int64_t r1, int64_t c0,
                           int64_t c1, int32_t thr, uint64_t* hist, uint64_t* pairs, int64_t cap,
                           uint64_t* cursor, cudaStream_t st) {
  ensure_pool_retained();
  const int64_t rows = r1 - r0, cols = c1 - c0;
  int64_t ccap = rows * cols;                 // upper bound on the range's pairs
  if (ccap > (1LL << 22)) ccap = 1LL << 22;
  if (const char* ev = getenv("PMH_ALLPAIRS_CCAP")) ccap = atoll(ev) > 0 ? atoll(ev) : 1;  // tests
  unsigned long long* tmp = nullptr;          // [zeros, ccursor, cand[ccap]]
  cudaError_t e = cudaMallocAsync((void**)&tmp, sizeof(unsigned long long) * (size_t)(ccap + 2), st);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  PMH_CUDA(cudaMemsetAsync(tmp, 0, 2 * sizeof(unsigned long long), st));
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, allpairs_lo_kernel, 256, 0);
  if (per_sm < 1) per_sm = 1;
  const int64_t ntiles = ((rows + AP_TILE - 1) / AP_TILE) * ((cols + AP_TILE - 1) / AP_TILE);
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > ntiles) grid = ntiles;
  allpairs_lo_kernel<<<(unsigned)grid, 256, 0, st>>>(sigs, m, r0, r1, c0, c1, tmp, tmp + 2, ccap,
                                                     tmp + 1);
  allpairs_cand_kernel<<<(unsigned)(sms * 8), 256, 0, st>>>(
      sigs, m, tmp + 2, ccap, tmp + 1, thr, (unsigned long long*)hist,
      (unsigned long long*)pairs, cap, (unsigned long long*)cursor);
  allpairs_zeros_kernel<<<1, 32, 0, st>>>(tmp, tmp + 1, ccap, (unsigned long long*)hist);
  PMH_CUDA(cudaGetLastError());
  const int rc = launch_allpairs_reduce(sigs, m, m, EqU64{}, r0, r1, c0, c1, thr, hist, pairs, cap,
                                        cursor, st, tmp + 1, (unsigned long long)ccap);
  cudaFreeAsync(tmp, st);
  return rc;
}
}  // namespace

extern "C" {

int pmh_allpairs_hist(const uint64_t* sigs, int64_t n, int64_t m, int64_t r0, int64_t r1,
                      int64_t c0, int64_t c1, int32_t thr, uint64_t* hist, uint64_t* pairs,
                      int64_t cap, uint64_t* cursor, void* stream) {
  if (m < 1 || m > 65535 || r0 < 0 || r1 > n || c0 < 0 || c1 > n || r0 > r1 || c0 > c1)
    return set_error(PMH_ERR_INVALID, "bad tile bounds");
  if (r0 == r1 || c0 == c1) return PMH_OK;
  // thr <= 0 lists every pair, zero counts included: single stage
  if (thr <= 0 || getenv("PMH_ALLPAIRS_1STAGE"))
    return launch_allpairs_reduce(sigs, m, m, EqU64{}, r0, r1, c0, c1, thr, hist, pairs, cap,
                                  cursor, (cudaStream_t)stream);
  return launch_allpairs_exact2(sigs, m, r0, r1, c0, c1, thr, hist, pairs, cap, cursor,
                                (cudaStream_t)stream);
}

// pmh_join.cuh: exact all-pairs histogram by a (component, value) hash join.
// Returns 1 (declined, nothing written) when the key lists exceed the work
// budget or thr <= 0; the caller then runs pmh_allpairs_hist.
__global__ void join_map_init_kernel(PairSlot* map, int64_t slots) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < slots;
       s += (int64_t)gridDim.x * blockDim.x) {
    map[s].key = PAIR_EMPTY;
    map[s].cnt = 0ULL;
  }
}

int pmh_allpairs_join_hist(const uint64_t* sigs, int64_t n, int64_t m, int64_t r0, int64_t r1,
                           int64_t c0, int64_t c1, int32_t thr, uint64_t* hist, uint64_t* pairs,
                           int64_t cap, uint64_t* cursor, int64_t max_visits, void* stream) {
  ensure_pool_retained();
  if (m < 1 || m > 65535 || r0 < 0 || r1 > n || c0 < 0 || c1 > n || r0 > r1 || c0 > c1)
    return set_error(PMH_ERR_INVALID, "bad tile bounds");
  if (n >= (1LL << 31)) return set_error(PMH_ERR_INVALID, "n must be < 2^31");
  if (r0 == r1 || c0 == c1) return PMH_OK;
  if (thr <= 0) return 1;   // zero-count pairs would have to be listed
  cudaStream_t st = (cudaStream_t)stream;
  int logC = 10;
  while ((1LL << logC) < 2 * n) logC++;
  const size_t per_comp = (sizeof(JoinSlot) + sizeof(int32_t)) << logC;
  const size_t budget = (size_t)1536 << 20;   // table memory per component group
  int64_t G = (int64_t)(budget / (per_comp + sizeof(int32_t) * (size_t)n));
  G = G < 1 ? 1 : (G > m ? m : G);
  const int64_t groups = (m + G - 1) / G;
  if (max_visits <= 0) max_visits = 1LL << 26;
  char* ws = nullptr;
  const size_t b_tab = sizeof(JoinSlot) * ((size_t)G << logC), b_head = sizeof(int32_t) * ((size_t)G << logC),
               b_next = sizeof(int32_t) * (size_t)n * (size_t)G;
  PMH_CUDA(cudaMallocAsync((void**)&ws, b_tab + b_head + b_next + 64, st));
  JoinSlot* tab = (JoinSlot*)ws;
  int32_t* head = (int32_t*)(ws + b_tab);
  int32_t* next = (int32_t*)(ws + b_tab + b_head);
  unsigned long long* ctr = (unsigned long long*)(ws + b_tab + b_head + b_next);   // visits, occ
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(sms * 8);
  auto build = [&](int64_t g) -> cudaError_t {
    const int64_t k0 = g * G, gg = (m - k0) < G ? (m - k0) : G;
    cudaError_t e = cudaMemsetAsync(tab, 0, sizeof(JoinSlot) * ((size_t)gg << logC), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(head, 0xFF, sizeof(int32_t) * ((size_t)gg << logC), st);
    if (e != cudaSuccess) return e;
    join_insert_kernel<<<grid, 256, 0, st>>>(sigs, n, m, k0, gg, tab, head, next, logC);
    return cudaGetLastError();
  };
  auto group_g = [&](int64_t g) { const int64_t k0 = g * G; return (m - k0) < G ? (m - k0) : G; };
  int rc = PMH_OK;
  cudaError_t e = cudaMemsetAsync(ctr, 0, 16, st);
  for (int64_t g = 0; g < groups && e == cudaSuccess; g++) {
    e = build(g);
    if (e == cudaSuccess) {
      join_emit_kernel<<<grid, 256, 0, st>>>(next, n, group_g(g), r0, r1, c0, c1, ctr, nullptr, 0);
      e = cudaGetLastError();
    }
  }
  unsigned long long visits = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&visits, ctr, 8, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) { cudaFreeAsync(ws, st); return cuda_fail(e, "join count"); }
  if ((long long)visits > max_visits) { cudaFreeAsync(ws, st); return 1; }
  int logM = 10;
  while ((1ULL << logM) < 2 * visits) logM++;
  PairSlot* map = nullptr;
  e = cudaMallocAsync((void**)&map, sizeof(PairSlot) << logM, st);
  if (e != cudaSuccess) { cudaFreeAsync(ws, st); return cuda_fail(e, "join map"); }
  join_map_init_kernel<<<grid, 256, 0, st>>>(map, 1LL << logM);
  for (int64_t g = 0; g < groups && e == cudaSuccess; g++) {
    if (groups > 1) e = build(g);   // one group: the tables of the count pass are still there
    if (e == cudaSuccess) {
      join_emit_kernel<<<grid, 256, 0, st>>>(next, n, group_g(g), r0, r1, c0, c1, nullptr, map, logM);
      e = cudaGetLastError();
    }
  }
  // pairs in range: a in [r0, r1), b in [c0, c1), b > a
  unsigned long long in_range = 0;
  for (int64_t a = r0; a < r1; a++) {
    const int64_t lo = c0 > a + 1 ? c0 : a + 1;
    if (c1 > lo) in_range += (unsigned long long)(c1 - lo);
  }
  if (e == cudaSuccess) {
    join_scan_kernel<<<grid, 256, 0, st>>>(map, 1LL << logM, m, thr, (unsigned long long*)hist,
                                           (unsigned long long*)pairs, cap,
                                           (unsigned long long*)cursor, ctr + 1);
    join_zeros_kernel<<<1, 1, 0, st>>>((unsigned long long*)hist, ctr + 1, in_range);
    e = cudaGetLastError();
  }
  cudaFreeAsync(map, st);
  cudaFreeAsync(ws, st);
  if (e != cudaSuccess) rc = cuda_fail(e, "join");
  return rc;
}

int64_t pmh_bbit_words(int64_t m, int b) {
  if (m < 1 || b < 1 || b > 16) return -1;
  const int64_t fpw = 64 / b;
  return (m + fpw - 1) / fpw;
}

int pmh_bbit_pack(const uint64_t* sig, int64_t nsets, int64_t m, int b, uint64_t* packed,
                  void* stream) {
  if (b < 1 || b > 16) return set_error(PMH_ERR_INVALID, "b must be in 1..16");
  if (m < 1 || nsets < 0) return set_error(PMH_ERR_INVALID, "bad sizes");
  const int64_t W = pmh_bbit_words(m, b);
  const int64_t total = nsets * W;
  if (total == 0) return PMH_OK;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  bbit_pack_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(sig, nsets, m, b, 64 / b,
                                                                       W, packed);
  PMH_CUDA(cudaGetLastError());
  return PMH_OK;
}

int pmh_allpairs_bbit_hist(const uint64_t* packed, int64_t n, int64_t m, int b, int64_t r0,
                           int64_t r1, int64_t c0, int64_t c1, int32_t thr, uint64_t* hist,
                           uint64_t* pairs, int64_t cap, uint64_t* cursor, void* stream) {
  if (b < 1 || b > 16) return set_error(PMH_ERR_INVALID, "b must be in 1..16");
  if (m < 1 || m > 65535 || r0 < 0 || r1 > n || c0 < 0 || c1 > n || r0 > r1 || c0 > c1)
    return set_error(PMH_ERR_INVALID, "bad tile bounds");
  if (r0 == r1 || c0 == c1) return PMH_OK;
  const int fpw = 64 / b;
  uint64_t H = 0, L = 0;
  for (int f = 0; f < fpw; f++) {
    H |= 1ULL << (f * b + b - 1);
    L |= ((1ULL << (b - 1)) - 1ULL) << (f * b);
  }
  const int64_t W = pmh_bbit_words(m, b);
  cudaStream_t st = (cudaStream_t)stream;
  switch (b) {
    case 1: return launch_allpairs_reduce(packed, W, m, BBitNeqT<1>{m}, r0, r1, c0, c1, thr, hist, pairs, cap, cursor, st);
    case 2: return launch_allpairs_reduce(packed, W, m, BBitNeqT<2>{m}, r0, r1, c0, c1, thr, hist, pairs, cap, cursor, st);
    case 4: return launch_allpairs_reduce(packed, W, m, BBitNeqT<4>{m}, r0, r1, c0, c1, thr, hist, pairs, cap, cursor, st);
    case 8: return launch_allpairs_reduce(packed, W, m, BBitNeqT<8>{m}, r0, r1, c0, c1, thr, hist, pairs, cap, cursor, st);
    case 16: return launch_allpairs_reduce(packed, W, m, BBitNeqT<16>{m}, r0, r1, c0, c1, thr, hist, pairs, cap, cursor, st);
    default: return launch_allpairs_reduce(packed, W, m, BBitNeq{L, H, m}, r0, r1, c0, c1, thr, hist, pairs, cap, cursor, st);
  }
}

int pmh_bbit(const uint64_t* sig, int64_t nsets, int64_t m, int b, int64_t* out,
             void* stream) {
  if (b < 1 || b > 16) return set_error(PMH_ERR_INVALID, "b must be in 1..16");
  if (m < 1 || nsets < 0) return set_error(PMH_ERR_INVALID, "bad sizes");
  const int64_t total = nsets * m;
  if (total == 0) return PMH_OK;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  bbit_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(sig, total, m, b, out);
  PMH_CUDA(cudaGetLastError());
  return PMH_OK;
}

int pmh_mse_cell(int algo, int64_t m, const double* wa, const double* wb, int64_t npairs,
                 uint64_t seed, int64_t s, int64_t* matches, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (npairs < 1 || !wa || !wb) return set_error(PMH_ERR_INVALID, "fixture needs >= 1 weight pair");
  if (s < 0) return set_error(PMH_ERR_INVALID, "negative pair count");
  int vrc = validate_sketch(algo, m, wa, 1);
  if (vrc != PMH_OK) return vrc;
  if (s == 0) return PMH_OK;
  if (!matches) return set_error(PMH_ERR_INVALID, "matches buffer required");
  // element ranks of each side (K:944-955: q order)
  std::vector<int32_t> ra((size_t)npairs), rb((size_t)npairs);
  int64_t na = 0, nb = 0;
  for (int64_t q = 0; q < npairs; q++) {
    if (!(wa[q] >= 0.0) || !(wb[q] >= 0.0) || !(wa[q] > 0.0 || wb[q] > 0.0))
      return set_error(PMH_ERR_INVALID, "each pair needs a positive coordinate and no negatives");
    ra[(size_t)q] = (int32_t)na;
    rb[(size_t)q] = (int32_t)nb;
    na += wa[q] > 0.0;
    nb += wb[q] > 0.0;
  }
  if (na == 0 || nb == 0) return set_error(PMH_ERR_EMPTY, "cannot sketch an empty set");
  // pairs per chunk: bound the device working set to ~512 MB
  const int64_t per_pair = 16 * (na + nb) + 16 * m + 28;
  int64_t C = (512LL << 20) / per_pair;
  C = C < 1 ? 1 : (C > s ? s : C);
  C = C > (1LL << 30) ? (1LL << 30) : C;
  if (const char* ev = getenv("PMH_MSE_CHUNK_PAIRS")) {  // test hook: force chunking
    const long long cap = atoll(ev);
    if (cap > 0 && cap < C) C = cap;
  }
  ensure_pool_retained();
  double *d_wa = nullptr, *d_wb = nullptr, *d_w = nullptr;
  int32_t *d_ra = nullptr, *d_rb = nullptr, *d_cnt = nullptr;
  uint64_t *d_ids = nullptr, *d_sig = nullptr;
  int64_t *d_off = nullptr, *d_match = nullptr, *d_status = nullptr;
  int rc = PMH_OK;
  auto alloc = [&](void** p, size_t bytes) {
    if (rc != PMH_OK) return;
    cudaError_t e = cudaMallocAsync(p, bytes, st);
    if (e != cudaSuccess) rc = set_error(PMH_ERR_NOMEM, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
  };
  alloc((void**)&d_wa, sizeof(double) * npairs);
  alloc((void**)&d_wb, sizeof(double) * npairs);
  alloc((void**)&d_ra, sizeof(int32_t) * npairs);
  alloc((void**)&d_rb, sizeof(int32_t) * npairs);
  alloc((void**)&d_ids, sizeof(uint64_t) * C * (na + nb));
  alloc((void**)&d_w, sizeof(double) * C * (na + nb));
  alloc((void**)&d_off, sizeof(int64_t) * (2 * C + 1));
  alloc((void**)&d_sig, sizeof(uint64_t) * 2 * C * m);
  alloc((void**)&d_cnt, sizeof(int32_t) * C);
  alloc((void**)&d_match, sizeof(int64_t) * s);
  alloc((void**)&d_status, 16);
  if (rc == PMH_OK) {
    cudaMemcpyAsync(d_wa, wa, sizeof(double) * npairs, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_wb, wb, sizeof(double) * npairs, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_ra, ra.data(), sizeof(int32_t) * npairs, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_rb, rb.data(), sizeof(int32_t) * npairs, cudaMemcpyHostToDevice, st);
    rc = pmh_status_reset(d_status, st);
  }
  for (int64_t t0 = 0; rc == PMH_OK && t0 < s; t0 += C) {
    const int64_t c = s - t0 < C ? s - t0 : C;
    MseGenArgs g{d_wa, d_wb, d_ra, d_rb, npairs, na, nb, seed, t0, c, d_ids, d_w, d_off};
    int64_t blocks = (c * npairs + 255) / 256;
    blocks = blocks < 1 ? 1 : (blocks > 148 * 16 ? 148 * 16 : blocks);
    mse_gen_kernel<<<(unsigned)blocks, 256, 0, st>>>(g);
    if (cudaGetLastError() != cudaSuccess) { rc = set_error(PMH_ERR_CUDA, "mse_gen_kernel launch"); break; }
    rc = pmh_sketch_csr_async(algo, m, d_ids, d_w, d_off, 2 * c, d_sig, nullptr, d_status, st);
    if (rc != PMH_OK) break;
    rc = pmh_count_equal(d_sig, d_sig + (size_t)c * m, c, m, d_cnt, st);
    if (rc != PMH_OK) break;
    int64_t wb_ = (c + 255) / 256;
    wb_ = wb_ > 148 * 16 ? 148 * 16 : wb_;
    widen_counts_kernel<<<(unsigned)wb_, 256, 0, st>>>(d_cnt, c, d_match + t0);
  }
  if (rc == PMH_OK) {
    int64_t err = -1;
    rc = pmh_status_check(d_status, &err, st);
  }
  if (rc == PMH_OK) {
    cudaError_t e = cudaMemcpyAsync(matches, d_match, sizeof(int64_t) * s, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) rc = set_error(PMH_ERR_CUDA, std::string("mse cell: ") + cudaGetErrorString(e));
  }
  void* bufs[] = {d_wa, d_wb, d_ra, d_rb, d_ids, d_w, d_off, d_sig, d_cnt, d_match, d_status};
  for (void* b : bufs)
    if (b) cudaFreeAsync(b, st);
  return rc;
}

int64_t pmh_parse_weighted_text(const char* buf, int64_t len, uint64_t* ids, double* weights,
                                int64_t cap) {
  if (!buf || len < 0 || cap < 0 || (cap > 0 && (!ids || !weights))) return -(int64_t(1) << 61);
  return pmh_ingest::parse_weighted_text(buf, len, ids, weights, cap);
}

int pmh_probe_pipe_peak(int kind, double* gops_out, double* ms_out) {
  if (kind < PROBE_LOP3 || kind > PROBE_FFMA) return set_error(PMH_ERR_INVALID, "unknown probe");
  int dev = 0, sms = 0;
  PMH_CUDA(cudaGetDevice(&dev));
  PMH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  uint32_t* d = nullptr;
  PMH_CUDA(cudaMalloc(&d, 16));
  cudaEvent_t a, b;
  PMH_CUDA(cudaEventCreate(&a));
  PMH_CUDA(cudaEventCreate(&b));
  // 8 CTAs x 256 threads per SM = full occupancy at <= 32 registers
  const int blocks = sms * 8, threads = 256;
  const int iters = kind == PROBE_DFMA ? 4096 : 16384;
  auto launch = [&](int it) {
    switch (kind) {
      case PROBE_LOP3: alu_probe_kernel<<<blocks, threads>>>(it, d); break;
      case PROBE_IMAD: imad_probe_kernel<<<blocks, threads>>>(it, d); break;
      case PROBE_DFMA: dfma_probe_kernel<<<blocks, threads>>>(it, d); break;
      default: ffma_probe_kernel<<<blocks, threads>>>(it, d); break;
    }
  };
  launch(256);  // warm-up
  float ms = 1e30f;
  for (int rep = 0; rep < 5; rep++) {  // best of 5 (clock ramp / co-tenant noise)
    PMH_CUDA(cudaEventRecord(a));
    launch(iters);
    PMH_CUDA(cudaEventRecord(b));
    PMH_CUDA(cudaEventSynchronize(b));
    float t = 0.f;
    PMH_CUDA(cudaEventElapsedTime(&t, a, b));
    ms = t < ms ? t : ms;
  }
  PMH_CUDA(cudaGetLastError());
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d);
  const double ops = (double)blocks * threads * iters * 16.0 * 8.0;   // thread-level ops
  if (gops_out) *gops_out = ops / (ms * 1e-3) / 1e9;
  if (ms_out) *ms_out = ms;
  return PMH_OK;
}

int pmh_math_eval(int fn, const double* x, int64_t n, double* out, void* stream) {
  if (fn < 0 || fn > 2 || n < 0)
    return set_error(PMH_ERR_INVALID, "fn must be 0 (log1p), 1 (expm1) or 2 (log1p, x = -U domain)");
  if (n == 0) return PMH_OK;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  math_eval_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(fn, x, n, out);
  PMH_CUDA(cudaGetLastError());
  return PMH_OK;
}

int pmh_probe_point_rate(int kind, double* gpts_out, double* ms_out) {
  if (kind < 0 || kind > 1) return set_error(PMH_ERR_INVALID, "kind must be 0 (log1p) or 1 (TruncExp)");
  int dev = 0, sms = 0;
  PMH_CUDA(cudaGetDevice(&dev));
  PMH_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  uint32_t* d = nullptr;
  PMH_CUDA(cudaMalloc(&d, 16));
  cudaEvent_t a, b;
  PMH_CUDA(cudaEventCreate(&a));
  PMH_CUDA(cudaEventCreate(&b));
  int per_sm = 1;
  auto kern = kind == 0 ? point_probe_kernel<0> : point_probe_kernel<1>;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
  const int blocks = sms * (per_sm > 0 ? per_sm : 1), threads = 256;
  const int iters = kind == 0 ? 2048 : 8192;
  kern<<<blocks, threads>>>(64, d);   // warm-up
  float ms = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    PMH_CUDA(cudaEventRecord(a));
    kern<<<blocks, threads>>>(iters, d);
    PMH_CUDA(cudaEventRecord(b));
    PMH_CUDA(cudaEventSynchronize(b));
    float t = 0.f;
    PMH_CUDA(cudaEventElapsedTime(&t, a, b));
    ms = t < ms ? t : ms;
  }
  PMH_CUDA(cudaGetLastError());
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d);
  if (gpts_out) *gpts_out = (double)blocks * threads * iters / (ms * 1e-3) / 1e9;
  if (ms_out) *ms_out = ms;
  return PMH_OK;
}

int pmh_probe_alu_peak(double* gops_out, double* ms_out) {
  return pmh_probe_pipe_peak(PROBE_LOP3, gops_out, ms_out);
}

}  // extern "C"

