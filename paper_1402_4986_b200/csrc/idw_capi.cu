// idw_capi.cu -- the extern "C" shim of libidw_b200.so (include/idw_b200.h).
//
// One call == one reference strategy call (strategies.py:148-261): validate the
// structural arguments, stage host buffers into HBM when the caller passed host
// memory, launch the variant kernel (+ the exact fix-up pass in FAST mode) on a
// per-device stream, and copy the predictions back.  No CPU fallback exists.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <string>

#include "idw_launch.h"

namespace idw {

// ===========================================================================
// MUFU roofline probe: independent rcp.approx chains, 8 per thread.
static __global__ void k_mufu_probe(float *out, int iters, unsigned long long *cycles) {
  float a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = 1.0f + 1e-3f * (threadIdx.x + k);
  long long c0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    // rcp then +1: not an involution, so ptxas cannot fold pairs of MUFU.RCP
    for (int k = 0; k < 8; ++k)
      asm volatile("{ rcp.approx.ftz.f32 %0, %0;\n\t add.ftz.f32 %0, %0, 0f3F800000; }" : "+f"(a[k]));
  }
  long long c1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.f) out[0] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cycles[0] = (unsigned long long)(c1 - c0);
}


static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }

static int bytes_per_point(int kind, int prec, int b) {
  const int e = prec == IDW_SINGLE ? 4 : 8;
  switch (kind) {
    case IDW_SOA: return e;
    case IDW_AOS: return 3 * e;
    case IDW_AOAS: return 4 * e;
    case IDW_SOAOS: return 16;
    case IDW_HYBRID: return b == 0 ? 16 : 8;
  }
  return 0;
}
static int nbuf_of(int kind) {
  return kind == IDW_SOA ? 3 : (kind == IDW_AOS || kind == IDW_AOAS) ? 1 : 2;
}

// device_ptrs: the store buffers are read in place by the kernels, so their
// alignment matters (host buffers are staged into a 256-byte-aligned arena).
// K2 and K3 FAST (k_nested_warps) stage tiles with cp.async.bulk, which needs
// a 16-byte-aligned source for every layout; the other kernels need 16 bytes
// where they issue vector loads (every layout but AoS, whose 12/24-byte
// records take scalar loads).
static int validate(const idw_store *s, const void *qx, const void *qy, int64_t m, const idw_params *p,
                    const void *out, bool device_ptrs) {
  if (!s || !p) return set_error("null store or params"), IDW_E_ARG;
  if (s->kind < 0 || s->kind > 4) return set_error("unknown layout kind"), IDW_E_ARG;
  if (s->precision != IDW_SINGLE && s->precision != IDW_DOUBLE) return set_error("unknown precision"), IDW_E_ARG;
  if (s->precision == IDW_SINGLE && (s->kind == IDW_SOAOS || s->kind == IDW_HYBRID))
    return set_error("layout requires double precision"), IDW_E_UNSUPPORTED;  // layouts.py:80-82
  if (s->count < 1) return set_error("no data points"), IDW_E_ARG;           // strategies.py:128-129
  if (s->nbuf != nbuf_of(s->kind)) return set_error("buffer count does not match layout"), IDW_E_ARG;
  for (int b = 0; b < s->nbuf; ++b) {
    if (!s->buf[b]) return set_error("null store buffer"), IDW_E_ARG;
    const int64_t need = s->count * (int64_t)bytes_per_point(s->kind, s->precision, b);
    if (s->nbytes[b] < need) return set_error("store buffer shorter than its shape"), IDW_E_ARG;
    if (device_ptrs && p) {
      const bool bulk = p->variant == IDW_TILED || (p->variant == IDW_NESTED_IMPROVED && p->mode == IDW_FAST);
      const int align = (s->kind == IDW_AOS && !bulk) ? (s->precision == IDW_SINGLE ? 4 : 8) : 16;
      if (((uintptr_t)s->buf[b]) % align != 0)
        return set_error("device store buffer not " + std::to_string(align) + "-byte aligned"), IDW_E_ARG;
    }
  }
  if (m < 0) return set_error("negative query count"), IDW_E_ARG;
  if (m > 0 && (!qx || !qy || !out)) return set_error("null query or output pointer"), IDW_E_ARG;
  if (!(p->p > 0)) return set_error("power p must be > 0"), IDW_E_ARG;          // core.py:43-44
  if (!(p->zero_eps >= 0)) return set_error("zero_eps must be >= 0"), IDW_E_ARG;  // core.py:45-46
  if (p->variant < IDW_NAIVE || p->variant > IDW_NESTED_IMPROVED) return set_error("unknown variant"), IDW_E_ARG;
  if (p->mode != IDW_EXACT && p->mode != IDW_FAST) return set_error("unknown mode"), IDW_E_ARG;
  if (p->group_size < 1) return set_error("group_size must be >= 1"), IDW_E_ARG;  // strategies.py:57-58
  if (p->tile_size < 1) return set_error("tile_size must be >= 1"), IDW_E_ARG;
  if (p->splits < 0) return set_error("splits must be >= 0"), IDW_E_ARG;
  if (p->ndevices < 0 || p->ndevices > IDW_MAX_DEVICES)
    return set_error("ndevices must be in [0, " + std::to_string(IDW_MAX_DEVICES) + "]"), IDW_E_ARG;
  return 0;
}

// The one device of a device-pointer call.
static int single_device(const idw_params *p) { return p->ndevices >= 1 ? p->devices[0] : p->device; }

static std::mutex g_mu;

int kernel_occupancy(const void *kern, int dev, int threads, int smem, int *occ) {
  struct Key {
    const void *k;
    int dev, threads, smem;
    bool operator<(const Key &o) const {
      return std::tie(k, dev, threads, smem) < std::tie(o.k, o.dev, o.threads, o.smem);
    }
  };
  static std::mutex mu;
  static std::map<Key, int> cache;
  const Key key{kern, dev, threads, smem};
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return *occ = it->second, 0;
  }
  {
    // the attribute is a per-kernel ceiling: only ever raise it, so a launch
    // shaped for more shared memory stays valid after a smaller query
    static std::map<std::pair<const void *, int>, int> ceiling;
    std::lock_guard<std::mutex> lk(mu);
    int &c = ceiling[{kern, dev}];
    if (smem > 48 * 1024 && smem > c) {
      IDW_CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      c = smem;
    }
  }
  int o = 0;
  IDW_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, threads, smem));
  std::lock_guard<std::mutex> lk(mu);
  cache[key] = o;
  *occ = o;
  return 0;
}
static cudaStream_t g_streams[64];
static int g_sms[64];

static int device_stream(int dev, cudaStream_t *st, int *sms) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    set_error("no CUDA device available (libidw_b200 has no CPU fallback)");
    return IDW_E_CUDA;
  }
  if (dev < 0 || dev >= ndev || dev >= 64) return set_error("device ordinal out of range"), IDW_E_ARG;
  IDW_CK(cudaSetDevice(dev));
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_streams[dev]) {
    IDW_CK(cudaStreamCreateWithFlags(&g_streams[dev], cudaStreamNonBlocking));
    IDW_CK(cudaDeviceGetAttribute(&g_sms[dev], cudaDevAttrMultiProcessorCount, dev));
    // Per-call scratch (flags, split partials, data box) comes from the
    // device's default stream-ordered pool.  With the default release
    // threshold (0) every synchronisation hands the pages back and the next
    // call re-maps them (measured ~ms per call at C1); keep them instead.
    const char *keep = getenv("IDW_POOL_KEEP");
    if (!keep || atoi(keep) != 0) {
      cudaMemPool_t pool;
      IDW_CK(cudaDeviceGetDefaultMemPool(&pool, dev));
      uint64_t thr = ~uint64_t(0);
      IDW_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
  }
  *st = g_streams[dev];
  *sms = g_sms[dev];
  return 0;
}

static void fill_launch(Launch &L, const idw_store *s, const void *const *bufs, const void *qx, const void *qy,
                        int64_t m, const idw_params *p, void *out) {
  L.kind = s->kind;
  L.prec = s->precision;
  L.mode = p->mode;
  L.variant = p->variant;
  L.p2 = (p->p == 2.0);  // kernels.scalar_args: fast = p == 2.0 (kernels.py:22)
  L.epsp = p->zero_eps > 0;
  for (int b = 0; b < 3; ++b) L.g.b[b] = (const unsigned char *)(b < s->nbuf ? bufs[b] : nullptr);
  L.n = s->count;
  L.qx = qx;
  L.qy = qy;
  L.m = m;
  L.eps = p->zero_eps;
  L.wexp = -p->p / 2.0;
  // FAST screen: inflate eps by 2^-16 relative so FMA-contracted d2 can never
  // hide an exact coincidence; the fix-up re-tests with IEEE d2.
  L.eps_flag = p->zero_eps * (1.0 + 1.0 / 65536.0);
  L.G = p->group_size;
  L.T = p->tile_size;
  L.splits = p->splits;
  L.out = out;
}

// Events bracketing the variant kernels and the fix-up pass of the last
// idw_run_device call on this thread (read back by idw_last_kernel_ms).
struct EvSet {
  cudaEvent_t a = nullptr, b = nullptr, c = nullptr;
};
static thread_local EvSet g_ev[64];
static thread_local int g_last_dev = -1;

// evflags: cudaEventRecordExternal when the stream is being captured into a
// graph (the records become timing-capable event nodes of the graph).
static int dispatch(Launch &L, const EvSet *ev = nullptr, unsigned evflags = cudaEventRecordDefault) {
  int rc = 0;
  if (ev) IDW_CK(cudaEventRecordWithFlags(ev->a, L.st, evflags));
  switch (L.variant) {
    case IDW_NAIVE: rc = launch_naive(L); break;
    case IDW_TILED: rc = launch_tiled(L); break;
    case IDW_NESTED_IMPROVED: rc = launch_nested(L); break;
    case IDW_NESTED_ORIGINAL: rc = launch_nested_orig(L); break;
    default: set_error("unknown variant"); return IDW_E_ARG;
  }
  if (rc) return rc;
  if (ev) IDW_CK(cudaEventRecordWithFlags(ev->b, L.st, evflags));
  if (needs_fixup(L)) rc = launch_fixup(L);
  if (rc) return rc;
  if (ev) IDW_CK(cudaEventRecordWithFlags(ev->c, L.st, evflags));
  return rc;
}

static void fill_stats(idw_stats *st, const Launch &L, const idw_params *p, int64_t n, int64_t m) {
  if (!st) return;
  st->kernel_launches = L.launches;
  st->merge_events = p->variant == IDW_NESTED_ORIGINAL ? m * ((n + p->group_size - 1) / p->group_size) : 0;
}

}  // namespace idw

// A captured idw_run_device call (include/idw_b200.h: idw_plan_*).
struct idw_plan {
  int dev = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  idw::EvSet ev;
  int64_t launches = 0;
};

using namespace idw;

extern "C" {

int idw_abi_version(void) { return IDW_ABI_VERSION; }

int idw_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

const char *idw_last_error(void) { return g_err.c_str(); }

static int run_device_multi(const idw_store *s, const void *qx, const void *qy, int64_t m, const idw_params *p,
                            void *out, cudaStream_t caller, idw_stats *stats);

int idw_run_device(const idw_store *s, const void *qx, const void *qy, int64_t m, const idw_params *p, void *out,
                   void *stream, idw_stats *stats) {
  g_err.clear();
  int rc = validate(s, qx, qy, m, p, out, true);
  if (rc) return rc;
  if (m == 0) return 0;
  if (p->ndevices > 1) return run_device_multi(s, qx, qy, m, p, out, (cudaStream_t)stream, stats);
  cudaStream_t dst;
  int sms;
  const int dev = single_device(p);
  if ((rc = device_stream(dev, &dst, &sms))) return rc;
  Launch L;
  fill_launch(L, s, s->buf, qx, qy, m, p, out);
  L.st = (cudaStream_t)stream;
  L.dev = dev;
  L.sms = sms;
  unsigned char *flags = nullptr;
  StreamFree free_flags;
  if (needs_fixup(L)) {
    IDW_CK(cudaMallocAsync((void **)&flags, (size_t)m, L.st));
    L.flags = flags;
    free_flags.p = flags;
    free_flags.st = L.st;
  }
  EvSet &ev = g_ev[dev];
  if (!ev.a) {
    IDW_CK(cudaEventCreate(&ev.a));
    IDW_CK(cudaEventCreate(&ev.b));
    IDW_CK(cudaEventCreate(&ev.c));
  }
  rc = dispatch(L, &ev);
  g_last_dev = rc == 0 ? dev : -1;
  fill_stats(stats, L, p, s->count, m);
  return rc;
}

// Query shard k of `slots`: contiguous, whole 256-query units (a multiple of
// every kernel's query group, so no group straddles two shards), sizes within
// one unit -- partition.shard_bounds(m, slots, k, 256).
static void shard_of(int64_t m, int slots, int k, int64_t *lo, int64_t *hi) {
  const int64_t A = 256, units = (m + A - 1) / A, base = units / slots, extra = units % slots;
  const int64_t lu = k * base + std::min<int64_t>(k, extra);
  const int64_t hu = lu + base + (k < extra ? 1 : 0);
  *lo = std::min<int64_t>(m, lu * A);
  *hi = std::min<int64_t>(m, hu * A);
}

// Stream of the k-th use of `dev` in one call (k = 0: the device's stream).
static int slot_stream(int dev, int k, cudaStream_t *st, int *sms) {
  int rc = device_stream(dev, st, sms);
  if (rc || k == 0) return rc;
  static cudaStream_t extra[64][IDW_MAX_DEVICES];
  std::lock_guard<std::mutex> lk(g_mu);
  if (!extra[dev][k]) IDW_CK(cudaStreamCreateWithFlags(&extra[dev][k], cudaStreamNonBlocking));
  *st = extra[dev][k];
  return 0;
}

// Peer access between every pair of distinct listed devices (NVLink when the
// pair has it; cudaMemcpyPeerAsync works either way).  Enabled once.
static void enable_peers(const int32_t *devs, int n) {
  static bool done[64][64];
  std::lock_guard<std::mutex> lk(g_mu);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const int a = devs[i], b = devs[j];
      if (a == b || done[a][b]) continue;
      done[a][b] = true;
      int ok = 0;
      if (cudaDeviceCanAccessPeer(&ok, a, b) == cudaSuccess && ok && cudaSetDevice(a) == cudaSuccess)
        cudaDeviceEnablePeerAccess(b, 0);  // AlreadyEnabled is fine
      cudaGetLastError();
    }
}

// One entry of a host call's device list: its stream, query shard and arena.
struct Slot {
  int dev = 0, sms = 0;
  cudaStream_t st = nullptr;
  int64_t lo = 0, hi = 0;
  unsigned char *arena = nullptr;
  size_t off[10] = {};
  cudaEvent_t have_data = nullptr, e0 = nullptr, e1 = nullptr;
  Launch L;
};

// Host-buffer path shared by idw_run (cast qx/qy given) and idw_run_xy (the
// reference's (m, 2) float64 query array, split + cast + checked on device),
// over one device or a device list driven from this one host thread:
//   A. per entry: stream, query shard, one stream-ordered arena
//   B. store: host -> devices[0], then a binomial broadcast tree of
//      cudaMemcpyPeerAsync (round r: entries [0, 2^r) feed [2^r, 2^(r+1)))
//   C. per entry: its query shard host -> device, kernels
//   D. per entry: predictions device -> its slice of the caller's `out` (pinned staging when <= 1 MB)
// B-C are asynchronous across entries; D comes after every entry's C was
// issued (a copy into pageable memory returns only when it is done).
static int run_host(const idw_store *s, const void *qx, const void *qy, const double *xy, int64_t m,
                    const idw_params *p, void *out, idw_stats *stats) {
  const int nslot = p->ndevices > 0 ? p->ndevices : 1;
  const int32_t *devs = p->ndevices > 0 ? p->devices : &p->device;
  const size_t esz = s->precision == IDW_SINGLE ? 4 : 8;
  Slot S[IDW_MAX_DEVICES];
  int rc = 0;
  // the caller's current device is restored on every exit (a device list
  // switches devices; the caller's framework may rely on its own setting)
  struct DeviceRestore {
    int dev = -1;
    DeviceRestore() {
      if (cudaGetDevice(&dev) != cudaSuccess) {
        dev = -1;
        cudaGetLastError();
      }
    }
    ~DeviceRestore() {
      if (dev >= 0) cudaSetDevice(dev);
    }
  } restore_device;
  // arenas and events go back on every exit, early error returns included
  struct Guard {
    Slot *S;
    int n = 0;
    bool sync = true;
    ~Guard() {
      for (int k = 0; k < n; ++k) {
        cudaSetDevice(S[k].dev);
        if (sync) cudaStreamSynchronize(S[k].st);
        if (S[k].arena) cudaFreeAsync(S[k].arena, S[k].st);
      }
      cudaGetLastError();
    }
  } guard{S};
  int uses[64] = {};
  for (int k = 0; k < nslot; ++k) {
    if (devs[k] < 0 || devs[k] >= 64) return set_error("device ordinal out of range"), IDW_E_ARG;
    Slot &sl = S[k];
    sl.dev = devs[k];
    if ((rc = slot_stream(sl.dev, uses[sl.dev]++, &sl.st, &sl.sms))) return rc;
    shard_of(m, nslot, k, &sl.lo, &sl.hi);
  }
  if (nslot > 1) enable_peers(devs, nslot);
  // per-(device, entry) events, created once per host thread
  static thread_local cudaEvent_t evs[64][IDW_MAX_DEVICES][3];
  for (int d = 0; d < 64; ++d) uses[d] = 0;
  for (int k = 0; k < nslot; ++k) {
    Slot &sl = S[k];
    IDW_CK(cudaSetDevice(sl.dev));
    cudaEvent_t *e = evs[sl.dev][uses[sl.dev]++];
    for (int i = 0; i < 3; ++i)
      if (!e[i]) IDW_CK(cudaEventCreate(&e[i]));
    sl.have_data = e[0];
    sl.e0 = e[1];
    sl.e1 = e[2];
  }

  // A. arenas: buffers (+64 B slack for the rounded-up bulk copy of the tail
  // tile), qx, qy, out, flags, fix-up counter, non-finite flag, raw xy pairs
  for (int k = 0; k < nslot; ++k) {
    Slot &sl = S[k];
    const size_t mk = (size_t)(sl.hi - sl.lo);
    size_t total = 0;
    auto take = [&](size_t bytes) {
      size_t o = total;
      total += (bytes + 255) & ~size_t(255);
      return o;
    };
    for (int b = 0; b < s->nbuf; ++b) sl.off[b] = take((size_t)s->nbytes[b] + 64);
    sl.off[3] = take(esz * mk);
    sl.off[4] = take(esz * mk);
    sl.off[5] = take(esz * mk);
    sl.off[6] = take(mk);
    sl.off[7] = take(16);  // fix-up count (u64) and non-finite flag (u32) share one 16-byte word pair
    sl.off[8] = sl.off[7] + 8;
    sl.off[9] = xy ? take(2 * sizeof(double) * mk) : 0;
    IDW_CK(cudaSetDevice(sl.dev));
    IDW_CK(cudaMallocAsync((void **)&sl.arena, total, sl.st));
    guard.n = k + 1;
  }

  // B. the store: one host->device copy, then the peer broadcast tree
  IDW_CK(cudaSetDevice(S[0].dev));
  for (int b = 0; b < s->nbuf; ++b)
    IDW_CK(cudaMemcpyAsync(S[0].arena + S[0].off[b], s->buf[b], (size_t)s->nbytes[b], cudaMemcpyHostToDevice,
                           S[0].st));
  IDW_CK(cudaEventRecord(S[0].have_data, S[0].st));
  for (int j = 1; j < nslot; ++j) {
    int top = 1;
    while (top * 2 <= j) top *= 2;
    const Slot &src = S[j - top];
    Slot &dst = S[j];
    IDW_CK(cudaSetDevice(dst.dev));
    IDW_CK(cudaStreamWaitEvent(dst.st, src.have_data, 0));
    for (int b = 0; b < s->nbuf; ++b)
      IDW_CK(cudaMemcpyPeerAsync(dst.arena + dst.off[b], dst.dev, src.arena + src.off[b], src.dev,
                                 (size_t)s->nbytes[b], dst.st));
    IDW_CK(cudaEventRecord(dst.have_data, dst.st));
  }

  // C. queries in, kernels
  for (int k = 0; k < nslot; ++k) {
    Slot &sl = S[k];
    const int64_t mk = sl.hi - sl.lo;
    if (mk == 0) continue;
    IDW_CK(cudaSetDevice(sl.dev));
    unsigned char *A = sl.arena;
    IDW_CK(cudaMemsetAsync(A + sl.off[7], 0, 16, sl.st));  // nfixed + bad
    if (xy) {
      IDW_CK(cudaMemcpyAsync(A + sl.off[9], xy + 2 * sl.lo, 2 * sizeof(double) * (size_t)mk,
                             cudaMemcpyHostToDevice, sl.st));
      if ((rc = split_queries((const double *)(A + sl.off[9]), mk, s->precision, A + sl.off[3], A + sl.off[4],
                              (unsigned int *)(A + sl.off[8]), sl.st, sl.sms)))
        return rc;
    } else {
      IDW_CK(cudaMemcpyAsync(A + sl.off[3], (const char *)qx + esz * sl.lo, esz * (size_t)mk,
                             cudaMemcpyHostToDevice, sl.st));
      IDW_CK(cudaMemcpyAsync(A + sl.off[4], (const char *)qy + esz * sl.lo, esz * (size_t)mk,
                             cudaMemcpyHostToDevice, sl.st));
    }
    const void *dbuf[3] = {nullptr, nullptr, nullptr};
    for (int b = 0; b < s->nbuf; ++b) dbuf[b] = A + sl.off[b];
    Launch &L = sl.L;
    fill_launch(L, s, dbuf, A + sl.off[3], A + sl.off[4], mk, p, A + sl.off[5]);
    L.st = sl.st;
    L.dev = sl.dev;
    L.sms = sl.sms;
    if (needs_fixup(L)) L.flags = A + sl.off[6];
    L.nfixed = (unsigned long long *)(A + sl.off[7]);
    IDW_CK(cudaEventRecord(sl.e0, sl.st));
    if ((rc = dispatch(L))) return rc;
    IDW_CK(cudaEventRecord(sl.e1, sl.st));
  }

  // D. predictions out, straight into each entry's slice of `out`
  // A small result (<= 1 MB) is staged through pinned memory: the copies
  // are then asynchronous (a copy into pageable memory blocks the host per
  // entry) and one host memcpy moves it into `out`.
  constexpr size_t STAGE = 1 << 20;
  static thread_local unsigned long long *ctr = nullptr;  // [IDW_MAX_DEVICES][2] counters + STAGE bytes, pinned
  if (!ctr) IDW_CK(cudaHostAlloc((void **)&ctr, 2 * sizeof(unsigned long long) * IDW_MAX_DEVICES + STAGE,
                                 cudaHostAllocPortable));
  char *const stage = (size_t)m * esz <= STAGE ? (char *)(ctr + 2 * IDW_MAX_DEVICES) : nullptr;
  for (int k = 0; k < nslot; ++k) {
    Slot &sl = S[k];
    const int64_t mk = sl.hi - sl.lo;
    if (mk == 0) continue;
    IDW_CK(cudaSetDevice(sl.dev));
    IDW_CK(cudaMemcpyAsync((stage ? stage : (char *)out) + esz * sl.lo, sl.arena + sl.off[5], esz * (size_t)mk,
                           cudaMemcpyDeviceToHost, sl.st));
    // both counters in one copy into pinned memory (truly asynchronous; two
    // pageable copies cost two blocking round trips per call)
    IDW_CK(cudaMemcpyAsync(ctr + 2 * k, sl.arena + sl.off[7], 16, cudaMemcpyDeviceToHost, sl.st));
  }
  float kms = 0.f;
  int64_t nfix = 0, launches = 0;
  unsigned int nonfinite = 0;
  for (int k = 0; k < nslot; ++k) {
    Slot &sl = S[k];
    IDW_CK(cudaSetDevice(sl.dev));
    IDW_CK(cudaStreamSynchronize(sl.st));
    if (sl.hi == sl.lo) continue;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, sl.e0, sl.e1) == cudaSuccess) kms = std::max(kms, ms);
    nfix += (int64_t)ctr[2 * k];
    nonfinite |= (unsigned int)ctr[2 * k + 1];
    launches += sl.L.launches;
  }
  guard.sync = false;
  if (stage) std::memcpy(out, stage, (size_t)m * esz);
  if (stats) {
    stats->kernel_ms = kms;
    stats->fixup_queries = nfix;
    stats->kernel_launches = launches;
    stats->merge_events = p->variant == IDW_NESTED_ORIGINAL ? m * ((s->count + p->group_size - 1) / p->group_size) : 0;
  }
  if (nonfinite) {
    set_error("invalid coordinate");  // core.ensure_finite (core.py:113-116)
    return IDW_E_NONFINITE;
  }
  return 0;
}

// Device-resident form over a device list: the store, queries and output live
// on devices[0] (the caller's stream belongs to it).  Entry k >= 1 gets the
// store through the same peer-copy broadcast tree, its query shard by a peer
// copy from devices[0], runs on its own stream, and its predictions go back
// into its slice of `out` by a peer copy -- the gather; entry 0 works in
// place.  Asynchronous: the entries start after the caller's stream reaches
// the call, and the caller's stream waits for all of them.
static int run_device_multi(const idw_store *s, const void *qx, const void *qy, int64_t m, const idw_params *p,
                            void *out, cudaStream_t caller, idw_stats *stats) {
  const int nslot = p->ndevices;
  const int32_t *devs = p->devices;
  const size_t esz = s->precision == IDW_SINGLE ? 4 : 8;
  const int dev0 = devs[0];
  struct DeviceRestore {
    int dev = -1;
    DeviceRestore() {
      if (cudaGetDevice(&dev) != cudaSuccess) {
        dev = -1;
        cudaGetLastError();
      }
    }
    ~DeviceRestore() {
      if (dev >= 0) cudaSetDevice(dev);
    }
  } restore_device;
  Slot S[IDW_MAX_DEVICES];
  int uses[64] = {};
  for (int k = 0; k < nslot; ++k) {
    if (devs[k] < 0 || devs[k] >= 64) return set_error("device ordinal out of range"), IDW_E_ARG;
    Slot &sl = S[k];
    sl.dev = devs[k];
    if (int rc = slot_stream(sl.dev, uses[sl.dev]++, &sl.st, &sl.sms)) return rc;
    shard_of(m, nslot, k, &sl.lo, &sl.hi);
  }
  if (nslot > 1) enable_peers(devs, nslot);
  // inputs ready on the caller's stream
  cudaEvent_t ready = nullptr;
  IDW_CK(cudaSetDevice(dev0));
  IDW_CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  IDW_CK(cudaEventRecord(ready, caller));
  cudaEvent_t have[IDW_MAX_DEVICES] = {}, done[IDW_MAX_DEVICES] = {};
  struct Events {
    cudaEvent_t *a, *b, r;
    int n;
    ~Events() {
      cudaEventDestroy(r);  // released once their recorded work completes
      for (int k = 0; k < n; ++k) {
        if (a[k]) cudaEventDestroy(a[k]);
        if (b[k]) cudaEventDestroy(b[k]);
      }
    }
  } ev_guard{have, done, ready, nslot};
  int64_t launches = 0;
  for (int k = 0; k < nslot; ++k) {
    Slot &sl = S[k];
    IDW_CK(cudaSetDevice(sl.dev));
    IDW_CK(cudaEventCreateWithFlags(&have[k], cudaEventDisableTiming));
    IDW_CK(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
    IDW_CK(cudaStreamWaitEvent(sl.st, ready, 0));
  }
  // A. per entry >= 1: an arena for the store copy, the query shard and the
  //    output shard; entry 0 reads and writes the caller's buffers in place
  for (int k = 0; k < nslot; ++k) {
    Slot &sl = S[k];
    IDW_CK(cudaSetDevice(sl.dev));
    const size_t mk = (size_t)(sl.hi - sl.lo);
    size_t total = 0;
    auto take = [&](size_t bytes) {
      size_t o = total;
      total += (bytes + 255) & ~size_t(255);
      return o;
    };
    for (int b = 0; b < s->nbuf; ++b) sl.off[b] = k ? take((size_t)s->nbytes[b] + 64) : 0;
    sl.off[3] = k ? take(esz * mk) : 0;
    sl.off[4] = k ? take(esz * mk) : 0;
    sl.off[5] = k ? take(esz * mk) : 0;
    sl.off[6] = take(mk);  // flags
    IDW_CK(cudaMallocAsync((void **)&sl.arena, total ? total : 256, sl.st));
  }
  // B. the store: devices[0] holds it; broadcast tree to the other entries
  IDW_CK(cudaSetDevice(S[0].dev));
  IDW_CK(cudaEventRecord(have[0], S[0].st));
  auto store_ptr = [&](int k, int b) -> unsigned char * {
    return k ? S[k].arena + S[k].off[b] : (unsigned char *)s->buf[b];
  };
  for (int j = 1; j < nslot; ++j) {
    int top = 1;
    while (top * 2 <= j) top *= 2;
    const int src = j - top;
    Slot &dst = S[j];
    IDW_CK(cudaSetDevice(dst.dev));
    IDW_CK(cudaStreamWaitEvent(dst.st, have[src], 0));
    for (int b = 0; b < s->nbuf; ++b)
      IDW_CK(cudaMemcpyPeerAsync(store_ptr(j, b), dst.dev, store_ptr(src, b), S[src].dev, (size_t)s->nbytes[b],
                                 dst.st));
    IDW_CK(cudaEventRecord(have[j], dst.st));
  }
  // C. queries in, kernels, predictions back (the gather), completion
  for (int k = 0; k < nslot; ++k) {
    Slot &sl = S[k];
    const int64_t mk = sl.hi - sl.lo;
    IDW_CK(cudaSetDevice(sl.dev));
    if (mk > 0) {
      const char *qxs = (const char *)qx + esz * sl.lo, *qys = (const char *)qy + esz * sl.lo;
      char *outs = (char *)out + esz * sl.lo;
      const void *dq[2] = {qxs, qys};
      void *dout = outs;
      if (k) {
        IDW_CK(cudaMemcpyPeerAsync(sl.arena + sl.off[3], sl.dev, qxs, dev0, esz * (size_t)mk, sl.st));
        IDW_CK(cudaMemcpyPeerAsync(sl.arena + sl.off[4], sl.dev, qys, dev0, esz * (size_t)mk, sl.st));
        dq[0] = sl.arena + sl.off[3];
        dq[1] = sl.arena + sl.off[4];
        dout = sl.arena + sl.off[5];
      }
      const void *dbuf[3] = {nullptr, nullptr, nullptr};
      for (int b = 0; b < s->nbuf; ++b) dbuf[b] = store_ptr(k, b);
      Launch &L = sl.L;
      fill_launch(L, s, dbuf, dq[0], dq[1], mk, p, dout);
      L.st = sl.st;
      L.dev = sl.dev;
      L.sms = sl.sms;
      if (needs_fixup(L)) L.flags = sl.arena + sl.off[6];
      if (int rc = dispatch(L)) {
        cudaFreeAsync(sl.arena, sl.st);
        for (int j = 0; j < nslot; ++j)
          if (j != k) {
            cudaSetDevice(S[j].dev);
            cudaFreeAsync(S[j].arena, S[j].st);
          }
        return rc;
      }
      launches += L.launches;
      if (k) IDW_CK(cudaMemcpyPeerAsync(outs, dev0, sl.arena + sl.off[5], sl.dev, esz * (size_t)mk, sl.st));
    }
    IDW_CK(cudaFreeAsync(sl.arena, sl.st));
    IDW_CK(cudaEventRecord(done[k], sl.st));
  }
  IDW_CK(cudaSetDevice(dev0));
  for (int k = 0; k < nslot; ++k) IDW_CK(cudaStreamWaitEvent(caller, done[k], 0));
  if (stats) {
    stats->kernel_launches = launches;
    stats->merge_events = p->variant == IDW_NESTED_ORIGINAL ? m * ((s->count + p->group_size - 1) / p->group_size) : 0;
  }
  return 0;
}

static void plan_free(idw_plan *pl) {
  if (!pl) return;
  if (pl->exec) cudaGraphExecDestroy(pl->exec);
  if (pl->graph) cudaGraphDestroy(pl->graph);
  if (pl->ev.a) cudaEventDestroy(pl->ev.a);
  if (pl->ev.b) cudaEventDestroy(pl->ev.b);
  if (pl->ev.c) cudaEventDestroy(pl->ev.c);
  delete pl;
}

int idw_plan_create(const idw_store *s, const void *qx, const void *qy, int64_t m, const idw_params *p, void *out,
                    idw_plan **plan) {
  g_err.clear();
  if (!plan) return set_error("null plan pointer"), IDW_E_ARG;
  *plan = nullptr;
  int rc = validate(s, qx, qy, m, p, out, true);
  if (rc) return rc;
  if (m == 0) return set_error("a plan needs at least one query"), IDW_E_ARG;
  if (p->ndevices > 1) return set_error("a plan runs on one device (ndevices <= 1)"), IDW_E_ARG;
  cudaStream_t dst;
  int sms;
  const int dev = single_device(p);
  if ((rc = device_stream(dev, &dst, &sms))) return rc;
  idw_plan *pl = new idw_plan();
  pl->dev = dev;
  cudaStream_t cap = nullptr;
  auto fail = [&](int code) {
    if (cap) {
      cudaGraph_t g = nullptr;
      cudaStreamEndCapture(cap, &g);  // abandon a half-built capture
      if (g) cudaGraphDestroy(g);
      cudaStreamDestroy(cap);
    }
    cudaGetLastError();
    plan_free(pl);
    return code;
  };
  if (cudaEventCreate(&pl->ev.a) || cudaEventCreate(&pl->ev.b) || cudaEventCreate(&pl->ev.c))
    return set_error("cudaEventCreate failed"), fail(IDW_E_CUDA);
  if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess)
    return set_error("cudaStreamCreate failed"), fail(IDW_E_CUDA);
  if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeRelaxed) != cudaSuccess)
    return set_error("cudaStreamBeginCapture failed"), fail(IDW_E_CUDA);
  Launch L;
  fill_launch(L, s, s->buf, qx, qy, m, p, out);
  L.st = cap;
  L.dev = dev;
  L.sms = sms;
  unsigned char *flags = nullptr;
  if (needs_fixup(L)) {
    if (cudaMallocAsync((void **)&flags, (size_t)m, cap) != cudaSuccess)
      return set_error("cudaMallocAsync (captured) failed"), fail(IDW_E_CUDA);
    L.flags = flags;
  }
  if ((rc = dispatch(L, &pl->ev, cudaEventRecordExternal))) return fail(rc);
  if (flags) cudaFreeAsync(flags, cap);
  cudaGraph_t g = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(cap, &g);
  cudaStreamDestroy(cap);
  cap = nullptr;
  if (ce != cudaSuccess || !g) return set_error(std::string("stream capture: ") + cudaGetErrorString(ce)), fail(IDW_E_CUDA);
  pl->graph = g;
  if (cudaGraphInstantiate(&pl->exec, g, 0) != cudaSuccess)
    return set_error("cudaGraphInstantiate failed"), fail(IDW_E_CUDA);
  // upload now so the first launch does not pay for it
  if (cudaGraphUpload(pl->exec, dst) != cudaSuccess || cudaStreamSynchronize(dst) != cudaSuccess)
    return set_error("cudaGraphUpload failed"), fail(IDW_E_CUDA);
  pl->launches = L.launches;
  *plan = pl;
  return 0;
}

int idw_plan_launch(idw_plan *pl, void *stream) {
  g_err.clear();
  if (!pl || !pl->exec) return set_error("null plan"), IDW_E_ARG;
  IDW_CK(cudaSetDevice(pl->dev));
  IDW_CK(cudaGraphLaunch(pl->exec, (cudaStream_t)stream));
  return 0;
}

int64_t idw_plan_launches(const idw_plan *pl) { return pl ? pl->launches : 0; }

int idw_plan_kernel_ms(idw_plan *pl, double *variant_ms, double *fixup_ms) {
  g_err.clear();
  if (!pl) return set_error("null plan"), IDW_E_ARG;
  IDW_CK(cudaSetDevice(pl->dev));
  IDW_CK(cudaEventSynchronize(pl->ev.c));
  float a = 0.f, b = 0.f;
  IDW_CK(cudaEventElapsedTime(&a, pl->ev.a, pl->ev.b));
  IDW_CK(cudaEventElapsedTime(&b, pl->ev.b, pl->ev.c));
  if (variant_ms) *variant_ms = a;
  if (fixup_ms) *fixup_ms = b;
  return 0;
}

void idw_plan_destroy(idw_plan *pl) {
  if (!pl) return;
  cudaSetDevice(pl->dev);
  plan_free(pl);
}

int idw_run(const idw_store *s, const void *qx, const void *qy, int64_t m, const idw_params *p, void *out,
            idw_stats *stats) {
  g_err.clear();
  int rc = validate(s, qx, qy, m, p, out, false);
  if (rc) return rc;
  if (m == 0) return 0;
  return run_host(s, qx, qy, nullptr, m, p, out, stats);
}

int idw_run_xy(const idw_store *s, const double *xy, int64_t m, const idw_params *p, void *out, idw_stats *stats) {
  g_err.clear();
  int rc = validate(s, xy, xy, m, p, out, false);
  if (rc) return rc;
  if (m == 0) return 0;
  return run_host(s, nullptr, nullptr, xy, m, p, out, stats);
}

// Shape check of a destination/source store against the layout table.
static int check_store_shape(const idw_store *s, const char *what) {
  if (!s) return set_error(std::string("null ") + what), IDW_E_ARG;
  if (s->kind < 0 || s->kind > 4 || (s->precision != IDW_SINGLE && s->precision != IDW_DOUBLE))
    return set_error(std::string(what) + ": unknown layout or precision"), IDW_E_ARG;
  if (s->precision == IDW_SINGLE && (s->kind == IDW_SOAOS || s->kind == IDW_HYBRID))
    return set_error("layout requires double precision"), IDW_E_UNSUPPORTED;
  if (s->count < 1) return set_error("no data points"), IDW_E_ARG;
  if (s->nbuf != nbuf_of(s->kind)) return set_error(std::string(what) + ": buffer count does not match layout"), IDW_E_ARG;
  for (int b = 0; b < s->nbuf; ++b) {
    if (!s->buf[b]) return set_error(std::string(what) + ": null buffer"), IDW_E_ARG;
    if (s->nbytes[b] < s->count * (int64_t)bytes_per_point(s->kind, s->precision, b))
      return set_error(std::string(what) + ": buffer shorter than its shape"), IDW_E_ARG;
  }
  return 0;
}

int idw_pack_device(const double *x, const double *y, const double *z, int64_t n, const idw_store *dst,
                    int device, void *stream) {
  g_err.clear();
  int rc = check_store_shape(dst, "destination");
  if (rc) return rc;
  if (!x || !y || !z) return set_error("null component array"), IDW_E_ARG;
  if (n != dst->count) return set_error("component length != store count"), IDW_E_ARG;
  cudaStream_t st;
  int sms;
  if ((rc = device_stream(device, &st, &sms))) return rc;
  unsigned char *d[3] = {(unsigned char *)dst->buf[0], (unsigned char *)dst->buf[1], (unsigned char *)dst->buf[2]};
  return pack_device(x, y, z, n, dst->kind, dst->precision, d, (cudaStream_t)stream, sms);
}

int idw_convert_device(const idw_store *src, const idw_store *dst, int device, void *stream) {
  g_err.clear();
  int rc = check_store_shape(src, "source");
  if (rc) return rc;
  if ((rc = check_store_shape(dst, "destination"))) return rc;
  if (src->precision != dst->precision) return set_error("conversion keeps the precision"), IDW_E_ARG;
  if (src->count != dst->count) return set_error("source and destination counts differ"), IDW_E_ARG;
  cudaStream_t st;
  int sms;
  if ((rc = device_stream(device, &st, &sms))) return rc;
  const unsigned char *s3[3] = {(const unsigned char *)src->buf[0], (const unsigned char *)src->buf[1],
                                (const unsigned char *)src->buf[2]};
  unsigned char *d3[3] = {(unsigned char *)dst->buf[0], (unsigned char *)dst->buf[1], (unsigned char *)dst->buf[2]};
  return convert_device(s3, src->kind, d3, dst->kind, src->precision, src->count, (cudaStream_t)stream, sms);
}

int idw_last_kernel_ms(double *variant_ms, double *fixup_ms) {
  g_err.clear();
  if (g_last_dev < 0) return set_error("no completed idw_run_device call on this thread"), IDW_E_ARG;
  EvSet &ev = g_ev[g_last_dev];
  IDW_CK(cudaSetDevice(g_last_dev));
  IDW_CK(cudaEventSynchronize(ev.c));
  float a = 0.f, b = 0.f;
  IDW_CK(cudaEventElapsedTime(&a, ev.a, ev.b));
  IDW_CK(cudaEventElapsedTime(&b, ev.b, ev.c));
  if (variant_ms) *variant_ms = a;
  if (fixup_ms) *fixup_ms = b;
  return 0;
}

int idw_mufu_peak(int device, double *rcp_per_s, double *sm_hz) {
  g_err.clear();
  cudaStream_t st;
  int sms, rc;
  if ((rc = device_stream(device, &st, &sms))) return rc;
  float *dout = nullptr;
  unsigned long long *dcyc = nullptr;
  IDW_CK(cudaMallocAsync((void **)&dout, 16, st));
  IDW_CK(cudaMallocAsync((void **)&dcyc, 16, st));
  // one resident wave: block 0's clock64 span then equals the kernel span
  int per_sm = 0;
  IDW_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mufu_probe, 256, 0));
  const int blocks = sms * (per_sm > 0 ? per_sm : 1), threads = 256, iters = 8192;
  cudaEvent_t e0, e1;
  IDW_CK(cudaEventCreate(&e0));
  IDW_CK(cudaEventCreate(&e1));
  k_mufu_probe<<<blocks, threads, 0, st>>>(dout, 256, dcyc);  // warm-up
  IDW_CK_LAUNCH();
  IDW_CK(cudaEventRecord(e0, st));
  k_mufu_probe<<<blocks, threads, 0, st>>>(dout, iters, dcyc);
  IDW_CK_LAUNCH();
  IDW_CK(cudaEventRecord(e1, st));
  unsigned long long cyc = 0;
  IDW_CK(cudaMemcpyAsync(&cyc, dcyc, sizeof(cyc), cudaMemcpyDeviceToHost, st));
  IDW_CK(cudaStreamSynchronize(st));
  float ms = 0.f;
  IDW_CK(cudaEventElapsedTime(&ms, e0, e1));
  const double ops = (double)blocks * threads * 8.0 * iters;
  if (rcp_per_s) *rcp_per_s = ops / (ms * 1e-3);
  if (sm_hz) *sm_hz = (double)cyc / (ms * 1e-3);
  cudaFreeAsync(dout, st);
  cudaFreeAsync(dcyc, st);
  cudaStreamSynchronize(st);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return 0;
}

}  // extern "C"
