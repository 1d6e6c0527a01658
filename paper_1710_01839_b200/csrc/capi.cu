// capi.cu -- the extern "C" boundary of libmpmm_cuda.so (include/mpmm_cuda.h).
//
// Replaces the reference's compiled kernel module (pkg/src/mpmm/_kernels.pyx,
// selected by backend.py:28-56): the eight range kernels keep their
// argument meaning on host pointers, and device-resident whole-GEMM /
// elementwise entry points serve the multiply/predict/tune layers.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mpmm_cuda.h"
#include "trace.h"
#include "kernels.h"

using namespace mpmm;

namespace mpmm {
cudaError_t strassen_run(int comps, int64_t cutoff, int tile, int64_t m, int64_t l, int64_t n,
                         const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                         int64_t ldc, int64_t* stats, cudaStream_t stream);
int rt_init(const int* devs, int ndev, std::string* err);
int rt_finalize();
int rt_gpus(int* ids, int cap);
int rt_gemm_host(int comps, int algo, int tile, int64_t cutoff, int64_t m, int64_t l, int64_t n,
                 const double* a, const double* b, double* c, int* nonfinite, double* device_ms,
                 int64_t panels, std::string* err);
int exact_gemm(int comps, int64_t m, int64_t l, int64_t n, const double* A, int64_t lda,
               const double* B, int64_t ldb, double* C, int64_t ldc, cudaStream_t s,
               std::string* err);
void exact_release();
}  // namespace mpmm

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(MPMM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CU(call)                                  \
  do {                                            \
    cudaError_t _e = (call);                      \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

bool dims_ok(int64_t m, int64_t l, int64_t n) {
  const int64_t lim = (int64_t)1 << 30;
  return m >= 0 && l >= 0 && n >= 0 && m < lim && l < lim && n < lim;
}

void tile_for(int64_t n_min, int* tile, int* super) {
  // n_min is the reference's cache block size (multiply.py:148-160).  On the
  // GPU it selects the CTA tile configuration; results never
  // depend on it.  `super` is kept in the ABI for table compatibility (1).
  *super = 1;
  if (const char* env = std::getenv("MPMM_FORCE_TILE")) {   // experiments only
    int t = std::atoi(env);
    if (t >= 0 && t < TILE_COUNT) {
      *tile = t;
      return;
    }
  }
  if (n_min <= 16) {
    *tile = TILE_16;
  } else if (n_min <= 32) {
    *tile = TILE_32;
  } else if (n_min <= 64) {
    *tile = TILE_LPT;
  } else if (n_min <= 128) {
    *tile = TILE_32x64;
  } else {
    *tile = TILE_64;
  }
}

// Every mirror product goes through the EFT-domain gate (domain.cuh):
// scan, then the DFMA launch or the Dekker launch, so results equal the
// reference's on every input.
cudaError_t gemm(int comps, const GemmArgs& g) { return gemm_checked(comps, g); }

// ---------------------------------------------------------------------------
// host-pointer protocol plumbing: per-thread streams, stream-ordered buffers
// ---------------------------------------------------------------------------

// One copy stream and one compute stream per (host thread, device), created
// on first use; the reference calls its kernels from a thread pool
// (multiply.py:99-112), so per-thread streams keep concurrent calls apart.
struct HostStreams {
  int device = -1;
  cudaStream_t copy = nullptr, comp = nullptr;
};
thread_local HostStreams g_hs;

cudaError_t host_streams(HostStreams** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (g_hs.device != dev) {
    g_hs.device = dev;
    if ((e = cudaStreamCreateWithFlags(&g_hs.copy, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&g_hs.comp, cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = retain_default_pool()) != cudaSuccess) return e;
  }
  *out = &g_hs;
  return cudaSuccess;
}

// Stream-ordered device buffer (memory-pool backed: no device-wide sync).
struct DevBuf {
  double* p = nullptr;
  cudaStream_t s = nullptr;
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  cudaError_t alloc(size_t doubles, cudaStream_t stream) {
    s = stream;
    return cudaMallocAsync(reinterpret_cast<void**>(&p),
                           doubles ? doubles * sizeof(double) : sizeof(double), stream);
  }
};

struct Event {
  cudaEvent_t e = nullptr;
  ~Event() {
    if (e) cudaEventDestroy(e);
  }
  cudaError_t make() { return cudaEventCreateWithFlags(&e, cudaEventDisableTiming); }
};

int block_cells_impl(int comps, int64_t n_min, int64_t cell0, int64_t cell1, int64_t m,
                     int64_t l, int64_t n, const double* A, int64_t lda, const double* B,
                     int64_t ldb, double* C, int64_t ldc, cudaStream_t stream) {
  if (n_min < 1) return fail(MPMM_ERR_ARG, "block size must be positive");
  if (m == 0 || n == 0 || cell1 <= cell0) return MPMM_OK;
  const int64_t nbc = (n + n_min - 1) / n_min;
  const int64_t nbr = (m + n_min - 1) / n_min;
  if (cell0 < 0 || cell1 > nbc * nbr) return fail(MPMM_ERR_ARG, "cell range out of bounds");
  int tile, super;
  tile_for(n_min, &tile, &super);
  // one domain scan of A and B covers every rectangle below
  const int* words = nullptr;
  if (l > 0) {
    cudaError_t e = domain_scan(comps, A, lda, (int)m, (int)l, B, ldb, (int)n, &words, stream);
    if (e != cudaSuccess) return cuda_fail(e, "block_cells domain scan");
  }
  // The flattened cell range [cell0, cell1) is at most three rectangles:
  // the tail of the first block row, whole block rows, the head of the last.
  auto rect = [&](int64_t r0, int64_t r1, int64_t c0, int64_t c1) -> int {
    r1 = r1 < m ? r1 : m;
    c1 = c1 < n ? c1 : n;
    if (r1 <= r0 || c1 <= c0) return MPMM_OK;
    GemmArgs g{ALGO_BLOCK, tile, (int)(r1 - r0), (int)(c1 - c0), (int)l,
               A + comps * (r0 * lda), lda, B + comps * c0, ldb,
               C + comps * (r0 * ldc + c0), ldc, 1, nullptr, stream};
    cudaError_t e = words ? gemm_gated(comps, g, words) : gemm(comps, g);
    return e == cudaSuccess ? MPMM_OK : cuda_fail(e, "block_cells launch");
  };
  const int64_t ib0 = cell0 / nbc, jb0 = cell0 % nbc;
  const int64_t ib1 = (cell1 - 1) / nbc, jb1 = (cell1 - 1) % nbc;
  int rc;
  if (ib0 == ib1) return rect(ib0 * n_min, (ib0 + 1) * n_min, jb0 * n_min, (jb1 + 1) * n_min);
  if ((rc = rect(ib0 * n_min, (ib0 + 1) * n_min, jb0 * n_min, n)) != MPMM_OK) return rc;
  if (ib1 > ib0 + 1 && (rc = rect((ib0 + 1) * n_min, ib1 * n_min, 0, n)) != MPMM_OK) return rc;
  return rect(ib1 * n_min, (ib1 + 1) * n_min, 0, (jb1 + 1) * n_min);
}

// ---------------------------------------------------------------------------
// Streamed host product: ONE GEMM launch whose CTAs consume k-panels as
// their H2D copies land, writing C straight into the caller's page-locked
// buffer.  The copy stream copies A/B panel by panel and after each sets
// the panel's ready flag with a 4-byte copy from page-locked memory (copy
// engine, no kernel, so the GEMM CTAs spinning on the flags can never
// block it); the GEMM (gemm_tiled, wait_k_panel) needs no event between the
// streams, so the only exposed copy is the first 64-column panel, there is
// one launch tail instead of one per panel, and C leaves over PCIe from the
// epilogues while later tiles compute.  Per element the k order is the
// same (bit-identical).  Used when A, B and C are page-locked; otherwise
// the panelled path below.
// ---------------------------------------------------------------------------

// Set when a streamed product timed out waiting for a panel (a tool that
// serialises kernels against the copy stream): later products take the
// panelled path.
std::atomic<bool> g_streamed_off{false};

// A page-locked 1: the source of every panel flag.  A 4-byte H2D copy
// from it runs on the copy engine, never on an SM, so the GEMM CTAs
// spinning on the flags cannot block it (a memset or a kernel could be).
const int* pinned_one() {
  if (g_streamed_off.load(std::memory_order_relaxed)) return nullptr;
  static int* one = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    if (const char* env = std::getenv("MPMM_HOST_STREAMED"))   // measurement knob: 0 = off
      if (env[0] == '0') return;
    int* p = nullptr;
    if (cudaHostAlloc(reinterpret_cast<void**>(&p), sizeof(int), cudaHostAllocDefault) ==
        cudaSuccess) {
      *p = 1;
      one = p;
    } else {
      cudaGetLastError();
    }
  });
  return one;
}

// page-locked host memory: its device alias (nullptr otherwise)
void* pinned_alias(const void* host) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, host) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

// k columns per streamed panel (MPMM_STREAM_PANEL: measurement knob, a
// multiple of 16)
int64_t stream_panel() {
  static const int64_t v = [] {
    int64_t p = 64;
    if (const char* env = std::getenv("MPMM_STREAM_PANEL")) {
      const int64_t q = std::atoll(env);
      if (q >= 16 && q % 16 == 0) p = q;
    }
    return p;
  }();
  return v;
}

// MPMM_OK, an error, or -1: not applicable (the caller takes the panelled path)
int host_rows_gemm_streamed(int comps, int tile, int64_t rows, int64_t l, int64_t n,
                            const double* a_rows, const double* b, double* c_rows,
                            int* nonfinite_host, HostStreams* hs) {
  const int* one = pinned_one();
  const int64_t kStreamPanel = stream_panel();
  if (one == nullptr || tile == TILE_LPT || l < 2 * kStreamPanel) return -1;
  if (pinned_alias(a_rows) == nullptr || pinned_alias(b) == nullptr) return -1;
  double* dCh = static_cast<double*>(pinned_alias(c_rows));
  if (dCh == nullptr) return -1;
  const size_t el = comps * sizeof(double);
  // Two streaming orders.  k-panels (64 columns of A and rows of B): every
  // tile consumes panel after panel, so only the first panel is exposed --
  // as long as all panels land within one wave of tiles.  For large
  // operands (>= 128 MiB) they do not (DD 8192^3: 2 GiB of H2D take ~40 ms,
  // one wave computes in ~7 ms), so A goes by row panels and B by column
  // panels in the order the grouped tile raster consumes them: the first
  // wave needs ~16 A and ~19 B panels (~140 MB) and later waves find theirs
  // already landed.
  int64_t tile_mb = 128;   // MPMM_STREAM_TILE_MB: the switch-over (tests, measurements)
  if (const char* env = std::getenv("MPMM_STREAM_TILE_MB")) tile_mb = std::atoll(env);
  const bool tile_mode = tile_mb >= 0 &&
                         static_cast<int64_t>((rows * l + l * n) * el) >= (tile_mb << 20);
  constexpr int64_t kRowsPerA = 64, kColsPerB = 128;
  Geometry geo{};
  if (tile_mode) {
    cudaError_t ge = comps == 2 ? dd_gemm_geometry(ALGO_BLOCK, tile, &geo)
                                : qd_gemm_geometry(ALGO_BLOCK, tile, &geo);
    if (ge != cudaSuccess) return cuda_fail(ge, "streamed product: tile geometry");
  }
  const int na = tile_mode ? static_cast<int>((rows + kRowsPerA - 1) / kRowsPerA) : 0;
  const int nb = tile_mode ? static_cast<int>((n + kColsPerB - 1) / kColsPerB) : 0;
  const int npan = tile_mode ? na + nb : static_cast<int>((l + kStreamPanel - 1) / kStreamPanel);
  DevBuf dA, dB, dflags;
  CU(dA.alloc(rows * l * comps, hs->comp));
  CU(dB.alloc(l * n * comps, hs->comp));
  // [0]: status (bit 0 non-finite, bit 2 panel wait timed out), [1 .. npan]:
  // panel flags; freed (stream-ordered) on every return path
  CU(dflags.alloc((npan + 2) / 2, hs->comp));
  int* dint = reinterpret_cast<int*>(dflags.p);
  CU(cudaMemsetAsync(dint, 0, (npan + 1) * sizeof(int), hs->comp));
  Event ready;
  CU(ready.make());
  CU(cudaEventRecord(ready.e, hs->comp));
  CU(cudaStreamWaitEvent(hs->copy, ready.e, 0));
  // The GEMM is enqueued FIRST: its CTAs start as soon as the flags are
  // zeroed and wait for each panel, so the copy/flag API calls below no
  // longer delay the launch.
  GemmArgs g{ALGO_BLOCK, tile, (int)rows, (int)n, (int)l, dA.p, l, dB.p, n, dCh, n, 0, dint,
             hs->comp};
  g.kready = dint + 1;
  if (tile_mode) {
    g.kpanel = 0;
    g.ktile_rows = static_cast<int>(kRowsPerA);
    g.ktile_cols = static_cast<int>(kColsPerB);
    g.ka_panels = na;
  } else {
    g.kpanel = static_cast<int>(kStreamPanel);
  }
  CU(gemm(comps, g));
  // the copies, each followed by its flag, in consumption order
  struct Copy { bool is_a; int64_t lo, hi; int flag; };
  std::vector<Copy> order;
  if (tile_mode) {
    const int first_group = static_cast<int>(
        std::min<int64_t>(na, (int64_t{kTileGroupM} * geo.bm + kRowsPerA - 1) / kRowsPerA));
    auto a_panel = [&](int q) {
      order.push_back({true, q * kRowsPerA, std::min<int64_t>(rows, (q + 1) * kRowsPerA), q});
    };
    for (int q = 0; q < first_group; ++q) a_panel(q);
    for (int q = 0; q < nb; ++q)
      order.push_back({false, q * kColsPerB, std::min<int64_t>(n, (q + 1) * kColsPerB), na + q});
    for (int q = first_group; q < na; ++q) a_panel(q);
  } else {
    for (int p = 0; p < npan; ++p)
      order.push_back({true, p * kStreamPanel, std::min<int64_t>(l, (p + 1) * kStreamPanel), p});
  }
  for (size_t i = 0; i < order.size(); ++i) {
    const Copy& c = order[i];
    cudaError_t e;
    if (!tile_mode) {              // k-panel: columns of A, rows of B
      e = cudaMemcpy2DAsync(dA.p + c.lo * comps, l * el, a_rows + c.lo * comps, l * el,
                            (c.hi - c.lo) * el, rows, cudaMemcpyHostToDevice, hs->copy);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(dB.p + c.lo * n * comps, b + c.lo * n * comps,
                            (c.hi - c.lo) * n * el, cudaMemcpyHostToDevice, hs->copy);
    } else if (c.is_a) {           // rows of A
      e = cudaMemcpyAsync(dA.p + c.lo * l * comps, a_rows + c.lo * l * comps,
                          (c.hi - c.lo) * l * el, cudaMemcpyHostToDevice, hs->copy);
    } else {                       // columns of B
      e = cudaMemcpy2DAsync(dB.p + c.lo * comps, n * el, b + c.lo * comps, n * el,
                            (c.hi - c.lo) * el, l, cudaMemcpyHostToDevice, hs->copy);
    }
    if (e != cudaSuccess) {
      // release the launched GEMM (it must not wait out its bound), then report
      for (size_t j = i; j < order.size(); ++j)
        cudaMemcpyAsync(dint + 1 + order[j].flag, one, sizeof(int), cudaMemcpyHostToDevice,
                        hs->copy);
      cudaStreamSynchronize(hs->comp);
      return cuda_fail(e, "streamed product: operand panel copy");
    }
    CU(cudaMemcpyAsync(dint + 1 + c.flag, one, sizeof(int), cudaMemcpyHostToDevice, hs->copy));
  }
  // The streamed launch runs the DFMA kernel before the operands have
  // landed, so their domain check (domain.cuh) follows the copies on the
  // copy stream, concurrent with the GEMM's tail.
  const int* words = nullptr;
  CU(domain_scan(comps, dA.p, l, (int)rows, (int)l, dB.p, n, (int)n, &words, hs->copy));
  int w[kDomainWords];
  CU(cudaMemcpyAsync(w, words, sizeof(w), cudaMemcpyDeviceToHost, hs->copy));
  int status = 0;   // pageable target: the copy completes before cudaMemcpyAsync returns
  CU(cudaMemcpyAsync(&status, dint, sizeof(int), cudaMemcpyDeviceToHost, hs->comp));
  CU(cudaStreamSynchronize(hs->copy));
  CU(cudaStreamSynchronize(hs->comp));
  if (status & 4) {
    // the panels never landed while the GEMM waited (its result is
    // incomplete): switch the process to the panelled path and let the
    // caller recompute with it
    g_streamed_off.store(true);
    return -1;
  }
  // operands outside the DFMA-exact domain: recompute C with the
  // reference's Dekker sequence (the rare path)
  if (domain_unsafe(w, 0, 0)) {
    CU(cudaMemsetAsync(dint, 0, sizeof(int), hs->comp));
    GemmArgs d{ALGO_BLOCK, tile, (int)rows, (int)n, (int)l, dA.p, l, dB.p, n, dCh, n, 0, dint,
               hs->comp};
    CU(comps == 2 ? dd_dekker_launch(d) : qd_dekker_launch(d));
    CU(cudaMemcpyAsync(&status, dint, sizeof(int), cudaMemcpyDeviceToHost, hs->comp));
    CU(cudaStreamSynchronize(hs->comp));
  }
  if (nonfinite_host) *nonfinite_host = status & 1;
  return MPMM_OK;
}

// rows x n block of C (host, row pitch n) = A rows (host, pitch l) * B
// (host, l x n), through the device, with the H2D of A and B split into
// k-panels on the copy stream so the GEMM of panel p overlaps the copy of
// panel p+1.  Each element's accumulator is carried through C between
// panels (bit-identical to one pass).  accumulate_c: start from C's value
// (block_cells semantics) instead of zero (simple_rows semantics).
int host_rows_gemm(int comps, int algo, int64_t n_min, int64_t rows, int64_t l, int64_t n,
                   const double* a_rows, const double* b, double* c_rows, bool accumulate_c,
                   int* nonfinite_host = nullptr) {
  if (nonfinite_host) *nonfinite_host = 0;
  if (rows == 0 || n == 0) return MPMM_OK;
  HostStreams* hs = nullptr;
  CU(host_streams(&hs));
  if (algo == ALGO_BLOCK && !accumulate_c) {
    int tile0 = TILE_16, super0 = 1;
    tile_for(n_min, &tile0, &super0);
    const int rc = host_rows_gemm_streamed(comps, tile0, rows, l, n, a_rows, b, c_rows,
                                           nonfinite_host, hs);
    if (rc != -1) return rc;
  }
  const size_t el = comps * sizeof(double);
  int* dflag = nullptr;
  if (nonfinite_host) {
    CU(cudaMallocAsync(reinterpret_cast<void**>(&dflag), sizeof(int), hs->comp));
    CU(cudaMemsetAsync(dflag, 0, sizeof(int), hs->comp));
  }
  DevBuf dA, dB, dC;
  CU(dA.alloc(rows * l * comps, hs->comp));
  CU(dB.alloc(l * n * comps, hs->comp));
  CU(dC.alloc(rows * n * comps, hs->comp));
  Event ready;                       // buffers allocated (stream-ordered on comp)
  CU(ready.make());
  CU(cudaEventRecord(ready.e, hs->comp));
  CU(cudaStreamWaitEvent(hs->copy, ready.e, 0));
  Event cin;
  CU(cin.make());
  if (accumulate_c) {
    CU(cudaMemcpyAsync(dC.p, c_rows, rows * n * el, cudaMemcpyHostToDevice, hs->copy));
    CU(cudaEventRecord(cin.e, hs->copy));
    CU(cudaStreamWaitEvent(hs->comp, cin.e, 0));
  }
  // up to 8 k-panels of >= 128: the first panel's copy is the only
  // exposed H2D; later copies hide under the previous panel's GEMM
  int64_t want = l >= 1024 ? 8 : (l >= 256 ? l / 128 : 1);
  if (const char* env = std::getenv("MPMM_HOST_PANELS")) {   // tuning knob
    int64_t v = std::atoll(env);
    if (v >= 1 && v <= 32) want = v < l ? v : (l > 0 ? l : 1);
  }
  // panel bounds: a short first panel (its H2D is the exposed one), the
  // rest of k in want - 1 equal panels
  std::vector<int64_t> kb{0};
  if (l > 0) {
    const int64_t step = (l + want - 1) / want;
    const int64_t first = want > 1 ? std::max<int64_t>(std::min<int64_t>(16, l), step / 4) : l;
    kb.push_back(first);
    const int64_t rest = l - first, np = want > 1 ? want - 1 : 0;
    for (int64_t q = 1; q <= np && rest > 0; ++q) {
      const int64_t b1 = first + (rest * q + np - 1) / np;
      if (b1 > kb.back()) kb.push_back(b1 < l ? b1 : l);
    }
    if (kb.back() != l) kb.push_back(l);
  }
  int tile = TILE_16, super = 1;
  if (algo != ALGO_SIMPLE) tile_for(n_min, &tile, &super);
  // The last panel runs in row slices so each slice's D2H (copy stream)
  // overlaps the next slice's GEMM; only the last slice's copy is exposed.
  int64_t nslice = rows >= 1024 ? 8 : (rows >= 512 ? 4 : (rows >= 256 ? 2 : 1));
  if (const char* env = std::getenv("MPMM_HOST_TAIL")) {     // tuning knob
    int64_t v = std::atoll(env);
    if (v >= 1 && v <= 8) nslice = v;
  }
  int64_t srows = ((rows + nslice - 1) / nslice + 63) / 64 * 64;
  const int npan = l > 0 ? static_cast<int>(kb.size()) - 1 : 1;
  std::vector<Event> ev(static_cast<size_t>(npan));
  std::vector<Event> sl(static_cast<size_t>(nslice));
  int64_t copied = 0;   // rows of C already queued for D2H
  for (int p = 0; p < npan; ++p) {
    const int64_t k0 = l > 0 ? kb[p] : 0, k1 = l > 0 ? kb[p + 1] : 0;
    if (l > 0) {
      CU(cudaMemcpy2DAsync(dA.p + k0 * comps, l * el, a_rows + k0 * comps, l * el,
                           (k1 - k0) * el, rows, cudaMemcpyHostToDevice, hs->copy));
      CU(cudaMemcpyAsync(dB.p + k0 * n * comps, b + k0 * n * comps, (k1 - k0) * n * el,
                         cudaMemcpyHostToDevice, hs->copy));
    }
    CU(ev[p].make());
    CU(cudaEventRecord(ev[p].e, hs->copy));
    CU(cudaStreamWaitEvent(hs->comp, ev[p].e, 0));
    const bool last = (k1 >= l);
    const int acc = (accumulate_c || p > 0) ? 1 : 0;
    // the panel's operands (every row slice below) in one domain scan
    const int* words = nullptr;
    if (algo != ALGO_BLOCK_FAST && k1 > k0)
      CU(domain_scan(comps, dA.p + k0 * comps, l, (int)rows, (int)(k1 - k0),
                     dB.p + k0 * n * comps, n, (int)n, &words, hs->comp));
    // the finite check only needs the final values: flag the last panel
    const int64_t sstep = last ? srows : rows;
    for (int64_t q0 = 0, si = 0; q0 < rows; q0 += sstep, ++si) {
      const int64_t q1 = q0 + sstep < rows ? q0 + sstep : rows;
      GemmArgs g{algo, tile, (int)(q1 - q0), (int)n, (int)(k1 - k0),
                 dA.p + (q0 * l + k0) * comps, l, dB.p + k0 * n * comps, n,
                 dC.p + q0 * n * comps, n, acc, last ? dflag : nullptr, hs->comp};
      CU(words ? gemm_gated(comps, g, words) : gemm(comps, g));
      if (last && q1 < rows) {   // this slice is final: copy it out under the next one
        CU(sl[si].make());
        CU(cudaEventRecord(sl[si].e, hs->comp));
        CU(cudaStreamWaitEvent(hs->copy, sl[si].e, 0));
        CU(cudaMemcpyAsync(c_rows + q0 * n * comps, dC.p + q0 * n * comps,
                           (q1 - q0) * n * el, cudaMemcpyDeviceToHost, hs->copy));
        copied = q1;
      }
    }
  }
  CU(cudaMemcpyAsync(c_rows + copied * n * comps, dC.p + copied * n * comps,
                     (rows - copied) * n * el, cudaMemcpyDeviceToHost, hs->comp));
  CU(cudaStreamSynchronize(hs->copy));
  if (dflag) {
    CU(cudaMemcpyAsync(nonfinite_host, dflag, sizeof(int), cudaMemcpyDeviceToHost, hs->comp));
    CU(cudaFreeAsync(dflag, hs->comp));
  }
  CU(cudaStreamSynchronize(hs->comp));
  return MPMM_OK;
}

int host_simple_rows(int comps, const double* a, const double* b, double* c, int64_t m,
                     int64_t l, int64_t n, int64_t i0, int64_t i1) {
  if (!dims_ok(m, l, n) || i0 < 0 || i1 > m) return fail(MPMM_ERR_ARG, "bad shape or row range");
  if (i1 <= i0 || n == 0) return MPMM_OK;
  return host_rows_gemm(comps, ALGO_SIMPLE, 0, i1 - i0, l, n, a + i0 * l * comps, b,
                        c + i0 * n * comps, false);
}

int host_block_cells(int comps, const double* a, const double* b, double* c, int64_t m,
                     int64_t l, int64_t n, int64_t n_min, int64_t cell0, int64_t cell1) {
  if (!dims_ok(m, l, n)) return fail(MPMM_ERR_ARG, "bad shape");
  if (n_min < 1) return fail(MPMM_ERR_ARG, "block size must be positive");
  if (m == 0 || n == 0 || cell1 <= cell0) return MPMM_OK;
  const int64_t nbc = (n + n_min - 1) / n_min;
  if (cell0 < 0 || cell1 > nbc * ((m + n_min - 1) / n_min))
    return fail(MPMM_ERR_ARG, "cell range out of bounds");
  const int64_t ib0 = cell0 / nbc, ib1 = (cell1 - 1) / nbc;
  const int64_t r0 = ib0 * n_min;
  const int64_t r1 = (ib1 + 1) * n_min < m ? (ib1 + 1) * n_min : m;
  const int64_t rows = r1 - r0;
  const int64_t ncells = nbc * ((m + n_min - 1) / n_min);
  if (cell0 % nbc == 0 && (cell1 % nbc == 0 || cell1 == ncells)) {
    // whole block rows: one pipelined pass over rows [r0, r1)
    return host_rows_gemm(comps, ALGO_BLOCK, n_min, rows, l, n, a + r0 * l * comps, b,
                          c + r0 * n * comps, true);
  }
  HostStreams* hs = nullptr;
  CU(host_streams(&hs));
  DevBuf dA, dB, dC;
  CU(dA.alloc(rows * l * comps, hs->comp));
  CU(dB.alloc(l * n * comps, hs->comp));
  CU(dC.alloc(rows * n * comps, hs->comp));
  const size_t el = comps * sizeof(double);
  CU(cudaMemcpyAsync(dA.p, a + r0 * l * comps, rows * l * el, cudaMemcpyHostToDevice, hs->comp));
  CU(cudaMemcpyAsync(dB.p, b, l * n * el, cudaMemcpyHostToDevice, hs->comp));
  CU(cudaMemcpyAsync(dC.p, c + r0 * n * comps, rows * n * el, cudaMemcpyHostToDevice, hs->comp));
  int rc = block_cells_impl(comps, n_min, cell0 - ib0 * nbc, cell1 - ib0 * nbc, rows, l, n, dA.p,
                            l, dB.p, n, dC.p, n, hs->comp);
  if (rc != MPMM_OK) return rc;
  // copy back ONLY the cells of [cell0, cell1): other threads of the
  // caller's pool own the rest of these block rows (multiply.py:99-112)
  auto back = [&](int64_t q0, int64_t q1, int64_t c0, int64_t c1) -> int {
    q1 = q1 < m ? q1 : m;
    c1 = c1 < n ? c1 : n;
    if (q1 <= q0 || c1 <= c0) return MPMM_OK;
    CU(cudaMemcpy2DAsync(c + (q0 * n + c0) * comps, n * el, dC.p + ((q0 - r0) * n + c0) * comps,
                         n * el, (c1 - c0) * el, q1 - q0, cudaMemcpyDeviceToHost, hs->comp));
    return MPMM_OK;
  };
  const int64_t jb0 = cell0 % nbc, jb1 = (cell1 - 1) % nbc;
  if (ib0 == ib1) {
    if ((rc = back(ib0 * n_min, (ib0 + 1) * n_min, jb0 * n_min, (jb1 + 1) * n_min)) != MPMM_OK)
      return rc;
  } else {
    if ((rc = back(ib0 * n_min, (ib0 + 1) * n_min, jb0 * n_min, n)) != MPMM_OK) return rc;
    if (ib1 > ib0 + 1 && (rc = back((ib0 + 1) * n_min, ib1 * n_min, 0, n)) != MPMM_OK) return rc;
    if ((rc = back(ib1 * n_min, (ib1 + 1) * n_min, 0, (jb1 + 1) * n_min)) != MPMM_OK) return rc;
  }
  CU(cudaStreamSynchronize(hs->comp));
  return MPMM_OK;
}

int host_ewise(int comps, int sign, const double* x, const double* y, double* out,
               int64_t rows, int64_t cols, int64_t i0, int64_t i1) {
  if (rows < 0 || cols < 0 || i0 < 0 || i1 > rows) return fail(MPMM_ERR_ARG, "bad row range");
  if (i1 <= i0 || cols == 0) return MPMM_OK;
  HostStreams* hs = nullptr;
  CU(host_streams(&hs));
  const int64_t r = i1 - i0, sz = r * cols * comps;
  DevBuf dX, dY;
  CU(dX.alloc(sz, hs->comp));
  CU(dY.alloc(sz, hs->comp));
  CU(cudaMemcpyAsync(dX.p, x + i0 * cols * comps, sz * sizeof(double), cudaMemcpyHostToDevice,
                     hs->comp));
  CU(cudaMemcpyAsync(dY.p, y + i0 * cols * comps, sz * sizeof(double), cudaMemcpyHostToDevice,
                     hs->comp));
  EwiseArgs e{comps, 1, (int)r, (int)cols, dX.p, cols, dY.p, cols, sign, nullptr, 0, 1,
              nullptr, 0, 1, dX.p, cols, hs->comp};
  CU(ewise_launch(e));
  CU(cudaMemcpyAsync(out + i0 * cols * comps, dX.p, sz * sizeof(double), cudaMemcpyDeviceToHost,
                     hs->comp));
  CU(cudaStreamSynchronize(hs->comp));
  return MPMM_OK;
}

}  // namespace

namespace mpmm {

cudaError_t retain_default_pool() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (e == cudaSuccess) e = cudaDeviceGetDefaultMemPool(&pool, dev);
  uint64_t keep = UINT64_MAX;
  if (e == cudaSuccess) e = cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  return e;
}

}  // namespace mpmm

extern "C" {

int mpmm_abi_version(void) { return MPMM_ABI_VERSION; }

const char* mpmm_last_error(void) { return g_err.c_str(); }

int mpmm_set_device(int device) {
  cudaError_t e = cudaSetDevice(device);
  return e == cudaSuccess ? MPMM_OK : cuda_fail(e, "cudaSetDevice");
}

int mpmm_device_count(int* count) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) {
    cudaGetLastError();
    c = 0;
  }
  *count = c;
  return MPMM_OK;
}

int mpmm_tile_for_nmin(int64_t n_min, int* tile, int* super_tiles) {
  if (n_min < 1) return fail(MPMM_ERR_ARG, "block size must be positive");
  tile_for(n_min, tile, super_tiles);
  return MPMM_OK;
}

int mpmm_gemm_geometry(int comps, int algo, int64_t n_min, int* tile_m, int* tile_n,
                       int* threads, int* ctas_per_sm, int* sm_count) {
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  int tile = TILE_16, super = 1;
  if (algo != MPMM_ALGO_SIMPLE) {
    if (n_min < 1) return fail(MPMM_ERR_ARG, "block size must be positive");
    tile_for(n_min, &tile, &super);
  }
  Geometry geo{0, 0, 0, 0};
  cudaError_t e = comps == 2 ? dd_gemm_geometry(algo, tile, &geo) : qd_gemm_geometry(algo, tile, &geo);
  if (e != cudaSuccess) return cuda_fail(e, "occupancy query");
  int dev = 0, sms = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  *tile_m = geo.bm;
  *tile_n = geo.bn;
  *threads = geo.threads;
  *ctas_per_sm = geo.ctas_per_sm;
  *sm_count = sms;
  return MPMM_OK;
}

int mpmm_dd_simple_rows(const double* a, const double* b, double* c, int64_t m, int64_t l,
                        int64_t n, int64_t i0, int64_t i1) {
  return host_simple_rows(2, a, b, c, m, l, n, i0, i1);
}
int mpmm_qd_simple_rows(const double* a, const double* b, double* c, int64_t m, int64_t l,
                        int64_t n, int64_t i0, int64_t i1) {
  return host_simple_rows(4, a, b, c, m, l, n, i0, i1);
}
int mpmm_dd_block_cells(const double* a, const double* b, double* c, int64_t m, int64_t l,
                        int64_t n, int64_t n_min, int64_t cell0, int64_t cell1) {
  return host_block_cells(2, a, b, c, m, l, n, n_min, cell0, cell1);
}
int mpmm_qd_block_cells(const double* a, const double* b, double* c, int64_t m, int64_t l,
                        int64_t n, int64_t n_min, int64_t cell0, int64_t cell1) {
  return host_block_cells(4, a, b, c, m, l, n, n_min, cell0, cell1);
}
int mpmm_dd_ewise_add(const double* x, const double* y, double* out, int64_t rows, int64_t cols,
                      int64_t i0, int64_t i1) {
  return host_ewise(2, 1, x, y, out, rows, cols, i0, i1);
}
int mpmm_dd_ewise_sub(const double* x, const double* y, double* out, int64_t rows, int64_t cols,
                      int64_t i0, int64_t i1) {
  return host_ewise(2, -1, x, y, out, rows, cols, i0, i1);
}
int mpmm_qd_ewise_add(const double* x, const double* y, double* out, int64_t rows, int64_t cols,
                      int64_t i0, int64_t i1) {
  return host_ewise(4, 1, x, y, out, rows, cols, i0, i1);
}
int mpmm_qd_ewise_sub(const double* x, const double* y, double* out, int64_t rows, int64_t cols,
                      int64_t i0, int64_t i1) {
  return host_ewise(4, -1, x, y, out, rows, cols, i0, i1);
}

int mpmm_gemm_host(int comps, int algo, int64_t n_min, int64_t m, int64_t l, int64_t n,
                   const double* a, const double* b, double* c, int accumulate, int* nonfinite) {
  TraceRange trace_("mpmm_gemm_host");
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (!dims_ok(m, l, n)) return fail(MPMM_ERR_ARG, "bad shape");
  if (algo != MPMM_ALGO_SIMPLE && algo != MPMM_ALGO_BLOCK && algo != MPMM_ALGO_BLOCK_FAST)
    return fail(MPMM_ERR_ARG, "bad algo");
  if (algo == MPMM_ALGO_BLOCK_FAST && comps != 2)
    return fail(MPMM_ERR_ARG, "the fast accuracy mode is implemented for DD only");
  if (algo != MPMM_ALGO_SIMPLE && n_min < 1) return fail(MPMM_ERR_ARG, "block size must be positive");
  return host_rows_gemm(comps, algo, n_min, m, l, n, a, b, c, accumulate != 0, nonfinite);
}

int mpmm_gemm_dev(int comps, int algo, int64_t n_min, int64_t m, int64_t l, int64_t n,
                  const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                  int64_t ldc, int accumulate, int* nonfinite, void* stream) {
  TraceRange trace_("mpmm_gemm_dev");
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (!dims_ok(m, l, n)) return fail(MPMM_ERR_ARG, "bad shape");
  if (lda < l || ldb < n || ldc < n) return fail(MPMM_ERR_ARG, "leading dimension too small");
  if (algo != MPMM_ALGO_SIMPLE && algo != MPMM_ALGO_BLOCK && algo != MPMM_ALGO_BLOCK_FAST)
    return fail(MPMM_ERR_ARG, "bad algo");
  if (algo == MPMM_ALGO_BLOCK_FAST && comps != 2)
    return fail(MPMM_ERR_ARG, "the fast accuracy mode is implemented for DD only");
  if (algo != MPMM_ALGO_SIMPLE && n_min < 1) return fail(MPMM_ERR_ARG, "block size must be positive");
  int tile = TILE_16, super = 1;
  if (algo != MPMM_ALGO_SIMPLE) tile_for(n_min, &tile, &super);
  GemmArgs g{algo, tile, (int)m, (int)n, (int)l, A, lda, B, ldb, C, ldc,
             accumulate ? 1 : 0, nonfinite, (cudaStream_t)stream};
  cudaError_t e = gemm(comps, g);
  return e == cudaSuccess ? MPMM_OK : cuda_fail(e, "gemm launch");
}

int mpmm_gemm_batched_dev(int comps, int algo, int64_t n_min, int64_t batch, int64_t m,
                          int64_t l, int64_t n, const void* problems, int accumulate,
                          int* nonfinite, void* stream) {
  TraceRange trace_("mpmm_gemm_batched_dev");
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (!dims_ok(m, l, n) || batch < 0 || batch > (1 << 24)) return fail(MPMM_ERR_ARG, "bad shape");
  if (algo != MPMM_ALGO_SIMPLE && algo != MPMM_ALGO_BLOCK && algo != MPMM_ALGO_BLOCK_FAST)
    return fail(MPMM_ERR_ARG, "bad algo");
  if (algo == MPMM_ALGO_BLOCK_FAST && comps != 2)
    return fail(MPMM_ERR_ARG, "the fast accuracy mode is implemented for DD only");
  if (algo != MPMM_ALGO_SIMPLE && n_min < 1) return fail(MPMM_ERR_ARG, "block size must be positive");
  if (batch == 0) return MPMM_OK;
  if (problems == nullptr) return fail(MPMM_ERR_ARG, "null problem array");
  int tile = TILE_16, super = 1;
  if (algo != MPMM_ALGO_SIMPLE) tile_for(n_min, &tile, &super);
  GemmArgs g{algo, tile, (int)m, (int)n, (int)l, nullptr, 0, nullptr, 0, nullptr, 0,
             accumulate ? 1 : 0, nonfinite, (cudaStream_t)stream};
  g.batch = (int)batch;
  g.probs = static_cast<const GemmProblem*>(problems);
  cudaError_t e = gemm(comps, g);
  return e == cudaSuccess ? MPMM_OK : cuda_fail(e, "batched gemm launch");
}

int mpmm_block_cells_dev(int comps, int64_t n_min, int64_t cell0, int64_t cell1, int64_t m,
                         int64_t l, int64_t n, const double* A, int64_t lda, const double* B,
                         int64_t ldb, double* C, int64_t ldc, void* stream) {
  TraceRange trace_("mpmm_block_cells_dev");
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (!dims_ok(m, l, n)) return fail(MPMM_ERR_ARG, "bad shape");
  return block_cells_impl(comps, n_min, cell0, cell1, m, l, n, A, lda, B, ldb, C, ldc,
                          (cudaStream_t)stream);
}

int mpmm_ewise_dev(int comps, int nops, int64_t rows, int64_t cols, const double* X,
                   int64_t ldx, const double* Y, int64_t ldy, int sy, const double* Z,
                   int64_t ldz, int sz, const double* W, int64_t ldw, int sw, double* O,
                   int64_t ldo, void* stream) {
  TraceRange trace_("mpmm_ewise_dev");
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (nops < 1 || nops > 3) return fail(MPMM_ERR_ARG, "nops must be 1..3");
  if (!dims_ok(rows, 0, cols)) return fail(MPMM_ERR_ARG, "bad shape");
  EwiseArgs e{comps, nops, (int)rows, (int)cols, X, ldx, Y, ldy, sy < 0 ? -1 : 1,
              Z, ldz, sz < 0 ? -1 : 1, W, ldw, sw < 0 ? -1 : 1, O, ldo, (cudaStream_t)stream};
  cudaError_t err = ewise_launch(e);
  return err == cudaSuccess ? MPMM_OK : cuda_fail(err, "ewise launch");
}

int mpmm_ewise_batched_dev(int comps, int64_t batch, int64_t rows, int64_t cols,
                           const void* problems, void* stream) {
  TraceRange trace_("mpmm_ewise_batched_dev");
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (!dims_ok(rows, 0, cols) || batch < 0 || batch > 65535) return fail(MPMM_ERR_ARG, "bad shape");
  if (batch == 0) return MPMM_OK;
  if (problems == nullptr) return fail(MPMM_ERR_ARG, "null problem array");
  cudaError_t err = ewise_batched_launch(comps, (int)batch, (int)rows, (int)cols,
                                         static_cast<const EwiseProblem*>(problems),
                                         (cudaStream_t)stream);
  return err == cudaSuccess ? MPMM_OK : cuda_fail(err, "batched ewise launch");
}

int mpmm_nonfinite_dev(int comps, int64_t rows, int64_t cols, const double* X, int64_t ldx,
                       int* flag, void* stream) {
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  cudaError_t err = nonfinite_launch(comps, X, ldx, (int)rows, (int)cols, flag,
                                     (cudaStream_t)stream);
  return err == cudaSuccess ? MPMM_OK : cuda_fail(err, "nonfinite launch");
}

int mpmm_exact_check_dev(int comps, int64_t m, int64_t l, int64_t n, const double* A,
                         int64_t lda, const double* B, int64_t ldb, const double* C, int64_t ldc,
                         const int64_t* idx_i, const int64_t* idx_j, int64_t count, int u_exp,
                         double* ratio, void* stream) {
  TraceRange trace_("mpmm_exact_check_dev");
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (!dims_ok(m, l, n) || count < 0) return fail(MPMM_ERR_ARG, "bad shape");
  cudaError_t err = exact_check_launch(comps, (int)l, A, lda, B, ldb, C, ldc, idx_i, idx_j, count,
                                       u_exp, ratio, (cudaStream_t)stream);
  return err == cudaSuccess ? MPMM_OK : cuda_fail(err, "exact check launch");
}

int mpmm_gen_inputs_dev(int comps, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                        uint64_t inc_lo, uint64_t first_draw, int64_t rows, int64_t cols,
                        double* out, void* stream) {
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (rows < 0 || cols < 0) return fail(MPMM_ERR_ARG, "bad shape");
  const int64_t count = rows * cols;
  if (count == 0) return MPMM_OK;
  cudaStream_t s = (cudaStream_t)stream;
  double* draws = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void**>(&draws), comps * count * sizeof(double), s));
  cudaError_t e = uniform_launch(state_hi, state_lo, inc_hi, inc_lo, first_draw, comps * count,
                                 draws, s);
  if (e == cudaSuccess) e = assemble_launch(comps, draws, count, out, s);
  cudaFreeAsync(draws, s);
  return e == cudaSuccess ? MPMM_OK : cuda_fail(e, "input generation launch");
}

int mpmm_oz_scan_dev(int by_cols, int comps, int64_t rows, int64_t cols, const double* X,
                     int64_t ld, int* EL, int* status, void* stream) {
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (!dims_ok(rows, 0, cols)) return fail(MPMM_ERR_ARG, "bad shape");
  cudaError_t e = oz_scan_launch(by_cols, X, ld, (int)rows, (int)cols, comps, EL, status,
                                 (cudaStream_t)stream);
  return e == cudaSuccess ? MPMM_OK : cuda_fail(e, "scan launch");
}

int mpmm_oz_residues_dev(int by_cols, int comps, int c0, int c1, int64_t rows, int64_t cols,
                         const double* X, int64_t ld, const int* shift, int nmod, int words,
                         int8_t* R, int64_t rpitch, int64_t rplane, void* stream) {
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (c0 < 0 || c1 > comps || c0 >= c1) return fail(MPMM_ERR_ARG, "bad component range");
  if (!dims_ok(rows, 0, cols) || nmod < 1 || nmod > 54) return fail(MPMM_ERR_ARG, "bad shape");
  if (words < 1 || words > 12) return fail(MPMM_ERR_ARG, "words must be 1..12");
  if (rpitch % 4) return fail(MPMM_ERR_ARG, "rpitch must be a multiple of 4");
  cudaError_t e = oz_residues_launch(by_cols, X, ld, (int)rows, (int)cols, comps, c0, c1, shift,
                                     nmod, words, R, rpitch, rplane, (cudaStream_t)stream);
  return e == cudaSuccess ? MPMM_OK : cuda_fail(e, "residues launch");
}

int mpmm_oz_plan(int comps, int64_t m, int64_t n, int64_t l, const int* ela, const int* elb,
                 int* njobs, int* jobs, int* na, int* ranges_a, int* shift_a, int* nb,
                 int* ranges_b, int* shift_b) {
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (m < 0 || n < 0 || l < 0) return fail(MPMM_ERR_ARG, "bad shape");
  int rc = oz_plan(comps, m, n, l, ela, elb, njobs, jobs, na, ranges_a, shift_a, nb, ranges_b,
                   shift_b);
  return rc == 0 ? MPMM_OK
                 : fail(MPMM_ERR_RANGE, "operand dynamic range too wide for the int8 CRT scheme");
}

int mpmm_gemm_exact_dev(int comps, int64_t m, int64_t l, int64_t n, const double* A,
                        int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                        void* stream) {
  TraceRange trace_("mpmm_gemm_exact_dev");
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (!dims_ok(m, l, n)) return fail(MPMM_ERR_ARG, "bad shape");
  if (lda < l || ldb < n || ldc < n) return fail(MPMM_ERR_ARG, "leading dimension too small");
  std::string err;
  const int rc = exact_gemm(comps, m, l, n, A, lda, B, ldb, C, ldc, (cudaStream_t)stream, &err);
  switch (rc) {
    case 0: return MPMM_OK;
    case 1: return fail(MPMM_ERR_ARG, err);
    case 4: return fail(MPMM_ERR_RANGE, err);
    case 5: return fail(MPMM_ERR_NONFINITE, err);
    default: return fail(MPMM_ERR_CUDA, err);
  }
}

int mpmm_residue_gemm_dev(int64_t m, int64_t n, int64_t k, int64_t batch, const int8_t* A,
                          const int8_t* Bt, uint8_t* R, void* stream) {
  TraceRange trace_("mpmm_residue_gemm_dev");
  if (!tc_residue_gemm_supported(m, n, k) || batch < 1 || batch > 54)
    return fail(MPMM_ERR_ARG, "residue GEMM needs m % 128 == 0, n % 256 == 0, k % 128 == 0, "
                              "k <= 131071, 1 <= batch <= 54");
  cudaError_t e = tc_residue_gemm(m, n, k, (int)batch, A, Bt, R, (cudaStream_t)stream);
  return e == cudaSuccess ? MPMM_OK : cuda_fail(e, "residue gemm launch");
}

int mpmm_exact_release(void) {
  exact_release();
  return MPMM_OK;
}

int mpmm_int8_gemm_batched_dev(int64_t m, int64_t n, int64_t k, int64_t batch, const int8_t* A,
                               const int8_t* Bt, int32_t* C, void* workspace, int64_t ws_bytes,
                               void* stream) {
  if (m % 16 || n % 16 || k % 16)
    return fail(MPMM_ERR_ARG, "int8 GEMM dimensions must be multiples of 16 (pad the operands)");
  std::string err;
  int rc = int8_gemm_batched(m, n, k, batch, A, Bt, C, workspace, (size_t)ws_bytes,
                             (cudaStream_t)stream, &err);
  return rc == 0 ? MPMM_OK : fail(rc == 1 ? MPMM_ERR_ARG : MPMM_ERR_CUDA, err);
}

int mpmm_oz_combine_dev(int comps, const void* jobs, int njobs, int64_t m, int64_t n, double* C,
                        int* status, void* stream) {
  TraceRange trace_("mpmm_oz_combine_dev");
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (njobs < 1 || njobs > 16 || !dims_ok(m, 0, n)) return fail(MPMM_ERR_ARG, "bad shape");
  cudaError_t e = oz_combine_launch(comps, jobs, njobs, (int)m, (int)n, C, status,
                                    (cudaStream_t)stream, false, 28);
  return e == cudaSuccess ? MPMM_OK : cuda_fail(e, "combine launch");
}

int mpmm_oz_shifts_dev(int comps, int nranges, const int* ranges, int64_t odim, const int* EL,
                       int* shift, int* beta, void* stream) {
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (nranges < 1 || nranges > 4 || odim < 0 || odim >= (1ll << 30))
    return fail(MPMM_ERR_ARG, "bad ranges or shape");
  for (int r = 0; r < nranges; ++r)
    if (ranges[2 * r] < 0 || ranges[2 * r + 1] > comps || ranges[2 * r] >= ranges[2 * r + 1])
      return fail(MPMM_ERR_ARG, "bad component range");
  cudaError_t e = oz_shifts_launch(comps, nranges, ranges, (int)odim, EL, shift, beta,
                                   (cudaStream_t)stream);
  return e == cudaSuccess ? MPMM_OK : cuda_fail(e, "shifts launch");
}

int mpmm_strassen_dev(int comps, int64_t cutoff, int64_t leaf_n_min, int64_t m, int64_t l,
                      int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                      double* C, int64_t ldc, int* nonfinite, int64_t* stats, void* stream) {
  TraceRange trace_("mpmm_strassen_dev");
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (!dims_ok(m, l, n)) return fail(MPMM_ERR_ARG, "bad shape");
  if (lda < l || ldb < n || ldc < n) return fail(MPMM_ERR_ARG, "leading dimension too small");
  if (cutoff < 2) return fail(MPMM_ERR_ARG, "Strassen cutoff must be >= 2");
  if (leaf_n_min < 1) return fail(MPMM_ERR_ARG, "leaf block size must be positive");
  if (stats) stats[0] = stats[1] = 0;
  int tile, super;
  tile_for(leaf_n_min, &tile, &super);
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = strassen_run(comps, cutoff, tile, m, l, n, A, lda, B, ldb, C, ldc, stats, s);
  if (e == cudaSuccess && nonfinite && m > 0 && n > 0)
    e = nonfinite_launch(comps, C, ldc, (int)m, (int)n, nonfinite, s);
  return e == cudaSuccess ? MPMM_OK : cuda_fail(e, "strassen");
}

int mpmm_init(int ngpus, const int* devices) {
  std::string err;
  int rc = rt_init(devices, ngpus, &err);
  return rc == 0 ? MPMM_OK : fail(rc, err);
}

int mpmm_finalize(void) { return rt_finalize(); }

int mpmm_runtime_gpus(int* ngpus, int* devices, int cap) {
  *ngpus = rt_gpus(devices, devices ? cap : 0);
  return MPMM_OK;
}

int mpmm_gemm_multi(int comps, int algo, int64_t n_min, int64_t cutoff, int64_t m, int64_t l,
                    int64_t n, const double* a, const double* b, double* c, int64_t panels,
                    int* nonfinite, double* device_ms) {
  TraceRange trace_("mpmm_gemm_multi");
  if (comps != 2 && comps != 4) return fail(MPMM_ERR_ARG, "comps must be 2 or 4");
  if (!dims_ok(m, l, n)) return fail(MPMM_ERR_ARG, "bad shape");
  if (algo < MPMM_ALGO_SIMPLE || algo > MPMM_ALGO_STRASSEN) return fail(MPMM_ERR_ARG, "bad algo");
  if (algo == MPMM_ALGO_BLOCK_FAST && comps != 2)
    return fail(MPMM_ERR_ARG, "the fast accuracy mode is implemented for DD only");
  if (algo != MPMM_ALGO_SIMPLE && n_min < 1) return fail(MPMM_ERR_ARG, "block size must be positive");
  if (algo == MPMM_ALGO_STRASSEN && cutoff < 2) return fail(MPMM_ERR_ARG, "Strassen cutoff must be >= 2");
  int tile = TILE_16, super = 1;
  if (algo != MPMM_ALGO_SIMPLE) tile_for(n_min, &tile, &super);
  std::string err;
  int rc = rt_gemm_host(comps, algo, tile, cutoff, m, l, n, a, b, c, nonfinite, device_ms, panels,
                        &err);
  return rc == 0 ? MPMM_OK : fail(rc, err);
}

struct MpmmTimer {
  cudaEvent_t start = nullptr, stop = nullptr;
};

int mpmm_timer_create(void** timer) {
  MpmmTimer* t = new MpmmTimer();
  cudaError_t e = cudaEventCreate(&t->start);
  if (e == cudaSuccess) e = cudaEventCreate(&t->stop);
  if (e != cudaSuccess) {
    if (t->start) cudaEventDestroy(t->start);
    delete t;
    return cuda_fail(e, "cudaEventCreate");
  }
  *timer = t;
  return MPMM_OK;
}

int mpmm_timer_start(void* timer, void* stream) {
  CU(cudaEventRecord(static_cast<MpmmTimer*>(timer)->start, (cudaStream_t)stream));
  return MPMM_OK;
}

int mpmm_timer_stop(void* timer, void* stream) {
  CU(cudaEventRecord(static_cast<MpmmTimer*>(timer)->stop, (cudaStream_t)stream));
  return MPMM_OK;
}

int mpmm_timer_elapsed_ms(void* timer, float* ms) {
  MpmmTimer* t = static_cast<MpmmTimer*>(timer);
  CU(cudaEventSynchronize(t->stop));
  CU(cudaEventElapsedTime(ms, t->start, t->stop));
  return MPMM_OK;
}

int mpmm_timer_destroy(void* timer) {
  MpmmTimer* t = static_cast<MpmmTimer*>(timer);
  if (t) {
    cudaEventDestroy(t->start);
    cudaEventDestroy(t->stop);
    delete t;
  }
  return MPMM_OK;
}

int mpmm_fp64_burn_dev(int op, int blocks, int threads, int64_t iters, double* scratch,
                       void* stream) {
  if (op != 0 && op != 1) return fail(MPMM_ERR_ARG, "op must be 0 (DFMA) or 1 (DADD)");
  cudaError_t err = fp64_burn_launch(op, blocks, threads, iters, scratch, (cudaStream_t)stream);
  return err == cudaSuccess ? MPMM_OK : cuda_fail(err, "fp64 burn launch");
}

}  // extern "C"
