// libhz C ABI (include/hz.h): contexts, tables, coefficient assembly, apply, batched BiCGSTAB,
// point sources; z-slab halo exchange and dot-product allreduce over NCCL for nranks > 1.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <condition_variable>
#include <map>
#include <queue>
#include <mutex>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "hz_debug.h"

#ifndef HZ_MG_BETA
#define HZ_MG_BETA 0.5   // complex shift of the multigrid preconditioner (reading A27)
#endif
#include "hz_internal.h"
#include "kernels.h"

// ---------------------------------------------------------------------------------------------
// errors and counters
// ---------------------------------------------------------------------------------------------
namespace hz {
static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
static std::atomic<long long> g_launches{0};
static inline void count_launch(long long n = 1) { g_launches += n; }
}  // namespace hz

using namespace hz;

#define HZ_CUDA(...)                                                                       \
  do {                                                                                     \
    cudaError_t e_ = (__VA_ARGS__);                                                        \
    if (e_ != cudaSuccess) {                                                               \
      set_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #__VA_ARGS__); \
      return e_ == cudaErrorMemoryAllocation ? HZ_ERR_OOM : HZ_ERR_CUDA;                    \
    }                                                                                      \
  } while (0)

#define HZ_TRY(...)                    \
  do {                                 \
    hz_status s_ = (__VA_ARGS__);      \
    if (s_ < 0) return s_;             \
  } while (0)

// ---------------------------------------------------------------------------------------------
// NCCL, loaded on demand (nranks > 1 only) so that libhz loads without NCCL on the path
// ---------------------------------------------------------------------------------------------
namespace {
struct Nccl {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
#define SYM(f) f = reinterpret_cast<decltype(f)>(dlsym(h, "nccl" #f))
    SYM(GetUniqueId); SYM(CommInitRank); SYM(CommDestroy); SYM(AllReduce); SYM(Broadcast);
    SYM(Send); SYM(Recv); SYM(GroupStart); SYM(GroupEnd); SYM(GetErrorString);
#undef SYM
    return GetUniqueId && CommInitRank && AllReduce && Send && Recv && GroupStart && GroupEnd;
  }
};
Nccl g_nccl;

hz_status nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return HZ_OK;
  set_error(std::string("NCCL error in ") + what + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
  return HZ_ERR_NCCL;
}

bool is_device_ptr(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Caching device allocator: blocks released by DBuf go to a free list and are reused by later
// requests of a similar size (assemble/solve per step would otherwise cudaMalloc/cudaFree ~8 fields
// per call, and cudaFree synchronises the device).  hz_trim_memory() returns the cache to CUDA.
// Blocks are keyed by (device, size): a block is only handed to a request on the device it was
// allocated on (the current device at the request, which every entry point sets from its context).
struct BlockCache {
  std::mutex m;
  std::multimap<std::pair<int, size_t>, void*> free;   // (device, size) -> block
  std::map<void*, std::pair<int, size_t>> info;          // block -> (device, size)
  cudaError_t acquire(size_t bytes, void** out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    {
      std::lock_guard<std::mutex> g(m);
      auto it = free.lower_bound({dev, bytes});
      if (it != free.end() && it->first.first == dev && it->first.second <= 2 * bytes + (1u << 20)) {
        *out = it->second;
        free.erase(it);
        return cudaSuccess;
      }
    }
    e = cudaMalloc(out, bytes);
    if (e == cudaErrorMemoryAllocation) {   // give the cache back and retry once
      cudaGetLastError();
      trim();
      e = cudaMalloc(out, bytes);
    }
    if (e == cudaSuccess) {
      std::lock_guard<std::mutex> g(m);
      info[*out] = {dev, bytes};
    }
    return e;
  }
  void release(void* p) {
    std::lock_guard<std::mutex> g(m);
    auto it = info.find(p);
    if (it == info.end()) return;
    free.emplace(it->second, p);
  }
  void trim() {
    std::lock_guard<std::mutex> g(m);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : free) {
      cudaSetDevice(kv.first.first);
      cudaFree(kv.second);
      info.erase(kv.second);
    }
    free.clear();
    cudaSetDevice(cur);
  }
};
BlockCache& cache() {
  static BlockCache* c = new BlockCache;   // never destroyed: blocks outlive static destructors
  return *c;
}

// RAII device buffer (cached)
struct DBuf {
  void* p = nullptr;
  size_t n = 0;
  ~DBuf() { if (p) cache().release(p); }
  cudaError_t ensure(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cache().release(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cache().acquire(bytes, &p);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
  template <typename T> T* as() const { return reinterpret_cast<T*>(p); }
};
}  // namespace

// ---------------------------------------------------------------------------------------------
// objects
// ---------------------------------------------------------------------------------------------
// Loopback communicator: P ranks of one process on one device (one host thread per rank), moving halo
// planes with one cudaMemcpyAsync per plane and summing the dots with a device kernel, behind the same
// call sites as NCCL.  Host barriers order the ranks' calls; GPU-side ordering goes through CUDA events
// (no kernel ever waits on another rank's kernel).
struct LoopGroup {
  int n = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  std::vector<void*> ptr;            // per rank: the buffer / field published for the current op
  std::vector<long long> nzl, fstride;
  std::vector<cudaEvent_t> ev, ev2;  // per rank: "published data ready", "done reading the others"
  std::vector<DBuf> tmp;             // per rank: reduction output before it overwrites the rank's buffer
  int refs = 0;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

struct hz_ctx {
  int device = 0, nranks = 1, rank = 0;
  ncclComm_t comm = nullptr;
  LoopGroup* loop = nullptr;   // loopback group (nranks > 1 without NCCL)
};

struct hz_table {
  Table t;
};

struct SolverWork {
  int nrhs = 0;
  DBuf rhat, p, v, t, r;        // fields [nrhs][nzl+2][ny][ldx]
  DBuf r1, r2;                  // BiCGStab(2) only
  DBuf xlo;                     // compensation term of the c64 iterate (double-float x)
  DBuf dotA, dotB, dotR, dotN, dotG;  // fp64 dot buffers
  DBuf state, active;
  DBuf partials, tickets;
  DBuf hb, hx;                  // staging for host b / x
  DBuf ph, sh;                  // right preconditioning: M⁻¹p, M⁻¹s
  struct MgDel {
    void operator()(MgHierarchy* m) const { mg_destroy(m); }
  };
  std::unique_ptr<MgHierarchy, MgDel> mg;   // complex shifted-Laplacian multigrid (precond = 1)
};

struct hz_coeffs {
  hz_ctx* ctx = nullptr;
  hz_dtype dtype = HZ_C64;
  hz_grid grid{};
  int ldx = 0;                 // row pitch of fields and model arrays (nx rounded up to 4)
  hz_mass mass = HZ_MASS_EQ8;
  hz_rule rule = HZ_RULE_GA;
  DBuf gam;                    // GAm: [5][nzl+2][ny][ldx] 27-node mean weights (t1, t2, mu0, mu1, mu2)
  double freq = 0, omega = 0, h = 0;
  double v_pml = 0;
  double vmin = 0, vmax = 0;   // the model's velocity range (all ranks)
  hz_pml pml{};
  Table table;                 // host copy actually used (rank 0's on all ranks)
  int n_g_dev = 0;             // rows uploaded (>= 2)
  double g_min = 0, g_max = 0, dg = 0;
  DBuf v;                      // [nzl+2][ny][ldx] R
  DBuf w;                      // [nzl+2][ny][ldx] R: 1/v² (the apply's model input)
  DBuf tab_f, tab_d;           // [n_g_dev][TAB_STRIDE] float / double rows (float only for C64)
  DBuf ctab_f, ctab_d;         // [n_g_dev][CTAB_STRIDE] pre-scaled class coefficients (apply)
  DBuf ctm_f;                  // [n_g_dev][TMTAB_STRIDE] the same with c0, m0 (complex64 tensor-map apply)
  DBuf pml_f[6], pml_d[6];     // dm x,y,z ; dp x,y,z (complex float / complex double)
  int lo[3], hi[3];
  int tab_lo = 0, tab_n = 2;   // table rows covering the model's G range (staged in smem by the apply)
  std::vector<std::complex<double>> am_h[3], ap_h[3];  // host copies for export
  DBuf partials, tickets;      // apply epilogue scratch
  int zc = 1, nchunks = 1;
  // complex64 tensor-map apply (apply27_tm): tile geometry, the map of w, cached maps of the fields
  // applied so far (keyed by pointer and RHS count), and per (RHS groups, RHS per CTA) a work list
  int tm_tx = 0, tm_ty = 0, tm_org = 0, tm_nval = 0;
  CUtensorMap tmap_w;
  std::map<std::pair<const void*, int>, CUtensorMap> tmap_u;
  struct TmPlan {
    DBuf work;
    int n_items = 0;
    int n_int = 0;  // halo-overlapped apply (nranks > 1): items [0, n_int) need no halo plane
    int grid = 1;   // resident CTAs: SMs × CTAs per SM
  };
  std::map<int, std::unique_ptr<TmPlan>> tm_plans;   // per RHS count
  DBuf tm_ctr;                 // apply27_tm work counter + CTA ticket
  // host-buffer applies: two copy streams and double-buffered device staging, so that the H2D copy of
  // one RHS group, the apply of the previous one and the D2H copy of the one before overlap
  struct HostIO {
    cudaStream_t in = nullptr, out = nullptr;
    cudaEvent_t start = nullptr, e_in[2] = {}, e_comp[2] = {}, e_out[2] = {};
    DBuf bin, bout;
    bool ok = false;
    cudaError_t init() {
      if (ok) return cudaSuccess;
      cudaError_t e = cudaStreamCreateWithFlags(&in, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
      for (int k = 0; k < 2 && e == cudaSuccess; k++) {
        e = cudaEventCreateWithFlags(&e_in[k], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&e_comp[k], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&e_out[k], cudaEventDisableTiming);
      }
      ok = e == cudaSuccess;
      return e;
    }
    ~HostIO() {
      if (in) cudaStreamDestroy(in);
      if (out) cudaStreamDestroy(out);
      for (cudaEvent_t ev : {start, e_in[0], e_in[1], e_comp[0], e_comp[1], e_out[0], e_out[1]})
        if (ev) cudaEventDestroy(ev);
    }
  };
  HostIO hio;
  // halo-overlapped apply (nranks > 1): the exchange runs on `cs` while the interior items run on the
  // caller's stream; `join` orders the boundary items after it
  struct Overlap {
    cudaStream_t cs = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    cudaError_t init() {
      if (cs) return cudaSuccess;
      cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
      return e;
    }
    ~Overlap() {
      if (cs) cudaStreamDestroy(cs);
      if (fork) cudaEventDestroy(fork);
      if (join) cudaEventDestroy(join);
    }
  };
  Overlap ovl;
  // visco-acoustic / variable-density medium (hz_coeffs_set_medium; readings A24, A25): every apply
  // goes through apply_medium.cu with b and κ⁻¹ = b/(v²(1 − i/(2Q))²), [nzl+2][ny][ldx] with halos
  bool medium = false;
  DBuf bmed, kinv;
  std::unique_ptr<SolverWork> work;
  size_t esz() const { return dtype == HZ_C64 ? 4 : 8; }   // real element size
  long long plane() const { return (long long)ldx * grid.ny; }
  long long fstride() const { return (long long)(grid.nz_local + 2) * plane(); }
  long long npoints() const { return (long long)grid.nx * grid.ny * grid.nz_local; }   // owned points
};
// internal helpers shared with the other translation units (hz_internal.h)
namespace hz {
void add_launches(long long n) { count_launch(n); }
bool device_pointer(const void* p) { return is_device_ptr(p); }
int ctx_device(const hz_ctx* c) { return c->device; }
}  // namespace hz

extern "C" {

const char* hz_last_error(void) { return g_err.c_str(); }
const char* hz_version(void) { return "libhz 0.2 (sm_100a)"; }
int hz_field_ldx(int nx) { return nx < 1 ? 0 : (nx + 3) & ~3; }
long long hz_kernel_launch_count(void) { return g_launches.load(); }
void hz_trim_memory(void) { cache().trim(); }

hz_status hz_get_unique_id(unsigned char id[128]) {
  if (!id) { set_error("hz_get_unique_id: id is NULL"); return HZ_ERR_INVALID_ARG; }
  if (!g_nccl.load()) { set_error("hz_get_unique_id: cannot load libnccl.so.2"); return HZ_ERR_NCCL; }
  ncclUniqueId u;
  HZ_TRY(nccl_check(g_nccl.GetUniqueId(&u), "ncclGetUniqueId"));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(id, &u, 128);
  return HZ_OK;
}

hz_status hz_ctx_create(int cuda_device, int nranks, int rank, const unsigned char* id, hz_ctx** out) {
  if (!out || nranks < 1 || rank < 0 || rank >= nranks) { set_error("hz_ctx_create: bad arguments"); return HZ_ERR_INVALID_ARG; }
  int ndev = 0;
  HZ_CUDA(cudaGetDeviceCount(&ndev));
  if (cuda_device < 0 || cuda_device >= ndev) { set_error("hz_ctx_create: bad device"); return HZ_ERR_INVALID_ARG; }
  HZ_CUDA(cudaSetDevice(cuda_device));
  std::unique_ptr<hz_ctx> c(new hz_ctx);
  c->device = cuda_device;
  c->nranks = nranks;
  c->rank = rank;
  if (nranks > 1) {
    if (!id) { set_error("hz_ctx_create: nranks > 1 needs a unique id"); return HZ_ERR_INVALID_ARG; }
    if (!g_nccl.load()) { set_error("hz_ctx_create: cannot load libnccl.so.2"); return HZ_ERR_NCCL; }
    ncclUniqueId u;
    memcpy(&u, id, 128);
    HZ_TRY(nccl_check(g_nccl.CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank"));
  }
  *out = c.release();
  return HZ_OK;
}

hz_status hz_ctx_create_loopback(int cuda_device, int nranks, hz_ctx** out) {
  if (!out || nranks < 1 || nranks > LOOP_MAX_RANKS) { set_error("hz_ctx_create_loopback: bad arguments (1..16 ranks)"); return HZ_ERR_INVALID_ARG; }
  int ndev = 0;
  HZ_CUDA(cudaGetDeviceCount(&ndev));
  if (cuda_device < 0 || cuda_device >= ndev) { set_error("hz_ctx_create_loopback: bad device"); return HZ_ERR_INVALID_ARG; }
  HZ_CUDA(cudaSetDevice(cuda_device));
  LoopGroup* g = new LoopGroup;
  g->n = nranks;
  g->ptr.assign(nranks, nullptr);
  g->nzl.assign(nranks, 0);
  g->fstride.assign(nranks, 0);
  g->ev.resize(nranks);
  g->ev2.resize(nranks);
  g->tmp.resize(nranks);
  for (int r = 0; r < nranks; r++) {
    HZ_CUDA(cudaEventCreateWithFlags(&g->ev[r], cudaEventDisableTiming));
    HZ_CUDA(cudaEventCreateWithFlags(&g->ev2[r], cudaEventDisableTiming));
  }
  g->refs = nranks;
  for (int r = 0; r < nranks; r++) {
    hz_ctx* c = new hz_ctx;
    c->device = cuda_device;
    c->nranks = nranks;
    c->rank = r;
    c->loop = nranks > 1 ? g : nullptr;
    out[r] = c;
  }
  if (nranks == 1) delete g;
  return HZ_OK;
}

void hz_ctx_destroy(hz_ctx* c) {
  if (!c) return;
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  if (c->loop) {
    LoopGroup* g = c->loop;
    bool last;
    {
      std::lock_guard<std::mutex> lk(g->m);
      last = --g->refs == 0;
    }
    if (last) {
      for (auto e : g->ev) cudaEventDestroy(e);
      for (auto e : g->ev2) cudaEventDestroy(e);
      delete g;
    }
  }
  delete c;
}

// ---------------------------------------------------------------------------------------------
// (1) weight table
// ---------------------------------------------------------------------------------------------
hz_status hz_build_weight_table(double g_min, double g_max, double dg, double lambda, const hz_angles* angles,
                                hz_table** out) {
  if (!out) { set_error("hz_build_weight_table: out is NULL"); return HZ_ERR_INVALID_ARG; }
  std::vector<double> th, ph;
  if (angles) {
    if (angles->n_theta < 1 || angles->n_phi < 1 || !angles->theta_rad || !angles->phi_rad) {
      set_error("hz_build_weight_table: bad angle grid");
      return HZ_ERR_INVALID_ARG;
    }
    th.assign(angles->theta_rad, angles->theta_rad + angles->n_theta);
    ph.assign(angles->phi_rad, angles->phi_rad + angles->n_phi);
  } else {
    for (int k = 0; k < 5; k++) {
      th.push_back(k * 10.0 * M_PI / 180.0);   // reading A10
      ph.push_back(k * 10.0 * M_PI / 180.0);
    }
  }
  std::unique_ptr<hz_table> t(new hz_table);
  HZ_TRY(build_table(g_min, g_max, dg, lambda, th, ph, &t->t));
  *out = t.release();
  return HZ_OK;
}

hz_status hz_table_import(double g_min, double dg, int n_g, const double* rows5, hz_table** out) {
  if (!out || !rows5 || n_g < 1 || !(dg > 0) || !std::isfinite(g_min)) {
    set_error("hz_table_import: bad arguments");
    return HZ_ERR_INVALID_ARG;
  }
  for (long long i = 0; i < 5LL * n_g; i++)
    if (!std::isfinite(rows5[i])) { set_error("hz_table_import: non-finite weight"); return HZ_ERR_DOMAIN; }
  std::unique_ptr<hz_table> t(new hz_table);
  t->t.g_min = g_min;
  t->t.dg = dg;
  t->t.n_g = n_g;
  t->t.rows5.assign(rows5, rows5 + 5LL * n_g);
  *out = t.release();
  return HZ_OK;
}

hz_status hz_table_rows(const hz_table* t, int* n_g, double* rows5, double* rows7) {
  if (!t) { set_error("hz_table_rows: NULL table"); return HZ_ERR_INVALID_ARG; }
  if (n_g) *n_g = t->t.n_g;
  for (int i = 0; i < t->t.n_g; i++) {
    const double* w = &t->t.rows5[5 * i];
    if (rows5) memcpy(rows5 + 5 * i, w, 5 * sizeof(double));
    if (rows7) {
      double* o = rows7 + 7 * i;
      o[0] = w[0];
      o[1] = w[1];
      o[2] = 1.0 - w[0] - w[1];           // ws3
      o[3] = w[2];                        // wm0 = mu0
      o[4] = 6.0 * w[3];                  // wm1 = 6 mu1 (A2)
      o[5] = 12.0 * w[4];                 // wm2 = 12 mu2
      o[6] = 1.0 - o[3] - o[4] - o[5];    // wm3
    }
  }
  return HZ_OK;
}

void hz_table_destroy(hz_table* t) { delete t; }

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// helpers on coeffs
// ---------------------------------------------------------------------------------------------
namespace {

// 1-D PML coefficients of one axis (A7, A8), in double on the host.
void pml_axis(int n, int npml, double h, double omega, double v_pml, double R,
              std::vector<std::complex<double>>& am, std::vector<std::complex<double>>& ap) {
  am.resize(n);
  ap.resize(n);
  auto gamma = [&](double s) {
    if (npml <= 0) return 0.0;
    const double L = npml * h;
    const double d = h * std::fmax(0.0, std::fmax(npml - s, s - (n - 1 - npml)));
    return 1.5 * v_pml / L * std::log(1.0 / R) * (d / L) * (d / L);
  };
  auto xi = [&](double s) { return std::complex<double>(1.0, gamma(s) / omega); };
  for (int i = 0; i < n; i++) {
    am[i] = 1.0 / (h * h * xi(i) * xi(i - 0.5));
    ap[i] = 1.0 / (h * h * xi(i) * xi(i + 0.5));
  }
}

// every entry point that launches work runs on its context's device
hz_status set_device(const hz_ctx* ctx) {
  if (cudaSetDevice(ctx->device) != cudaSuccess) {
    cudaGetLastError();
    set_error("cudaSetDevice failed");
    return HZ_ERR_CUDA;
  }
  return HZ_OK;
}

// R: arithmetic type, S: storage type (= the coeffs' dtype)
template <typename R, typename S = R>
ApplyParams<R, S> make_params(const hz_coeffs* c) {
  typedef typename Cx<R>::T C;
  ApplyParams<R, S> p;
  memset(&p, 0, sizeof(p));
  p.nx = c->grid.nx;
  p.ny = c->grid.ny;
  p.ldx = c->ldx;
  p.nzl = c->grid.nz_local;
  p.z0 = c->grid.z0;
  p.nzg = c->grid.nz_global;
  p.plane = c->plane();
  p.fstride = c->fstride();
  p.zc = c->zc;
  p.nchunks = c->nchunks;
  p.tm_tx = c->tm_tx;
  p.tm_ty = c->tm_ty;
  p.tm_org = c->tm_org;
  p.v = c->v.as<S>();
  p.w = c->w.as<S>();
  p.gam = c->rule != HZ_RULE_GA ? c->gam.as<S>() : nullptr;
  p.tab = sizeof(R) == 4 ? c->tab_f.as<R>() : c->tab_d.as<R>();
  p.ctab = sizeof(R) == 4 ? c->ctab_f.as<R>() : c->ctab_d.as<R>();
  p.ctm = sizeof(R) == 4 ? c->ctm_f.as<float>() : nullptr;
  p.tab_lo = c->tab_lo;
  p.tab_n = c->tab_n;
  p.invih2 = (R)(c->h * c->h);
  p.inv2ih2 = (R)(c->h * c->h / 2.0);
  p.inv3ih2 = (R)(c->h * c->h / 3.0);
  p.n_g = c->n_g_dev;
  p.g_min = (R)c->g_min;
  p.g_max = (R)c->g_max;
  p.inv_dg = (R)(1.0 / c->dg);
  p.inv_fh = (R)(1.0 / (c->freq * c->h));
  p.ih2 = (R)(1.0 / (c->h * c->h));
  p.w2 = (R)(c->omega * c->omega);
  for (int a = 0; a < 3; a++) {
    p.dm[a] = sizeof(R) == 4 ? c->pml_f[a].as<C>() : c->pml_d[a].as<C>();
    p.dp[a] = sizeof(R) == 4 ? c->pml_f[3 + a].as<C>() : c->pml_d[3 + a].as<C>();
    p.lo[a] = c->lo[a];
    p.hi[a] = c->hi[a];
  }
  return p;
}

// ---- communication: NCCL (one process per GPU) or the loopback group; no-ops for one rank ----
// Exchange the boundary planes of `field` ([nrhs][nzl+2][ny][ldx] complex) with the z neighbours.
hz_status halo_exchange(const hz_coeffs* c, void* field, int nrhs, size_t elem_bytes, cudaStream_t s) {
  const hz_ctx* ctx = c->ctx;
  if (ctx->nranks == 1) return HZ_OK;
  const size_t pb = (size_t)c->plane() * elem_bytes;
  const int nzl = c->grid.nz_local;
  char* base = reinterpret_cast<char*>(field);
  if (ctx->loop) {
    LoopGroup* g = ctx->loop;
    const int r = ctx->rank;
    g->ptr[r] = field;
    g->nzl[r] = nzl;
    g->fstride[r] = c->fstride();
    HZ_CUDA(cudaEventRecord(g->ev[r], s));
    g->barrier();
    for (int q : {r - 1, r + 1})
      if (q >= 0 && q < g->n) HZ_CUDA(cudaStreamWaitEvent(s, g->ev[q], 0));
    for (int k = 0; k < nrhs; k++) {
      char* f = base + (size_t)k * (size_t)c->fstride() * elem_bytes;
      if (r > 0) {   // halo plane 0 ← the lower neighbour's last owned plane
        const char* src = reinterpret_cast<const char*>(g->ptr[r - 1]) + (size_t)k * (size_t)g->fstride[r - 1] * elem_bytes;
        HZ_CUDA(cudaMemcpyAsync(f, src + (size_t)g->nzl[r - 1] * pb, pb, cudaMemcpyDeviceToDevice, s));
      }
      if (r < g->n - 1) {   // halo plane nzl+1 ← the upper neighbour's first owned plane
        const char* src = reinterpret_cast<const char*>(g->ptr[r + 1]) + (size_t)k * (size_t)g->fstride[r + 1] * elem_bytes;
        HZ_CUDA(cudaMemcpyAsync(f + (size_t)(nzl + 1) * pb, src + pb, pb, cudaMemcpyDeviceToDevice, s));
      }
    }
    HZ_CUDA(cudaEventRecord(g->ev2[r], s));
    g->barrier();
    for (int q : {r - 1, r + 1})   // the neighbours have read my boundary planes before I change them
      if (q >= 0 && q < g->n) HZ_CUDA(cudaStreamWaitEvent(s, g->ev2[q], 0));
    return HZ_OK;
  }
  HZ_TRY(nccl_check(g_nccl.GroupStart(), "ncclGroupStart"));
  for (int r = 0; r < nrhs; r++) {
    char* f = base + (size_t)r * (size_t)c->fstride() * elem_bytes;
    if (ctx->rank > 0) {
      g_nccl.Send(f + 1 * pb, pb, ncclChar, ctx->rank - 1, ctx->comm, s);
      g_nccl.Recv(f + 0 * pb, pb, ncclChar, ctx->rank - 1, ctx->comm, s);
    }
    if (ctx->rank < ctx->nranks - 1) {
      g_nccl.Send(f + (size_t)nzl * pb, pb, ncclChar, ctx->rank + 1, ctx->comm, s);
      g_nccl.Recv(f + (size_t)(nzl + 1) * pb, pb, ncclChar, ctx->rank + 1, ctx->comm, s);
    }
  }
  HZ_TRY(nccl_check(g_nccl.GroupEnd(), "ncclGroupEnd"));
  return HZ_OK;
}

// in-place allreduce of n doubles (op 0 = sum, 1 = max) over the ranks
hz_status comm_allreduce(const hz_ctx* ctx, double* buf, size_t n, int op, cudaStream_t s) {
  if (ctx->nranks == 1) return HZ_OK;
  if (ctx->loop) {
    LoopGroup* g = ctx->loop;
    const int r = ctx->rank;
    g->ptr[r] = buf;
    HZ_CUDA(g->tmp[r].ensure(n * sizeof(double)));
    HZ_CUDA(cudaEventRecord(g->ev[r], s));
    g->barrier();
    LoopPtrs lp;
    for (int q = 0; q < g->n; q++) {
      if (q != r) HZ_CUDA(cudaStreamWaitEvent(s, g->ev[q], 0));
      lp.p[q] = reinterpret_cast<const double*>(g->ptr[q]);
    }
    HZ_CUDA(launch_loop_reduce(lp, g->n, g->tmp[r].as<double>(), (long long)n, op, s));
    count_launch();
    HZ_CUDA(cudaEventRecord(g->ev2[r], s));
    g->barrier();
    for (int q = 0; q < g->n; q++)   // every rank has read my buffer before it is overwritten
      if (q != r) HZ_CUDA(cudaStreamWaitEvent(s, g->ev2[q], 0));
    HZ_CUDA(cudaMemcpyAsync(buf, g->tmp[r].p, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    return HZ_OK;
  }
  return nccl_check(g_nccl.AllReduce(buf, buf, n, ncclDouble, op == 0 ? ncclSum : ncclMax, ctx->comm, s), "ncclAllReduce");
}

hz_status allreduce_sum(const hz_coeffs* c, double* buf, size_t n, cudaStream_t s) {
  return comm_allreduce(c->ctx, buf, n, 0, s);
}

// broadcast n doubles of rank 0's buffer to every rank
hz_status comm_bcast(const hz_ctx* ctx, double* buf, size_t n, cudaStream_t s) {
  if (ctx->nranks == 1) return HZ_OK;
  if (ctx->loop) {
    LoopGroup* g = ctx->loop;
    const int r = ctx->rank;
    g->ptr[r] = buf;
    HZ_CUDA(cudaEventRecord(g->ev[r], s));
    g->barrier();
    if (r != 0) {
      HZ_CUDA(cudaStreamWaitEvent(s, g->ev[0], 0));
      HZ_CUDA(cudaMemcpyAsync(buf, g->ptr[0], n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    HZ_CUDA(cudaEventRecord(g->ev2[r], s));
    g->barrier();
    if (r == 0)
      for (int q = 1; q < g->n; q++) HZ_CUDA(cudaStreamWaitEvent(s, g->ev2[q], 0));
    return HZ_OK;
  }
  return nccl_check(g_nccl.Broadcast(buf, buf, n, ncclDouble, 0, ctx->comm, s), "ncclBroadcast");
}

// ---------------------------------------------------------------------------------------------
// complex64 tensor-map apply (apply27_tm): tile geometry, tensor maps, work lists
// ---------------------------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

hz_status tm_encoder() {
  if (g_encode) return HZ_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || fn == nullptr) {
    cudaGetLastError();
    set_error("cuTensorMapEncodeTiled is not available from the CUDA driver");
    return HZ_ERR_CUDA;
  }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return HZ_OK;
}

// Tile geometry: tile i computes the columns [i·tx − 1, (i+1)·tx − 1) (apply27_tm.cuh); ntx tiles of
// tx ∈ {32, 64} columns cover the pitched row (the pad columns too, which the apply writes as zeros):
// the width with the fewest box columns ntx·(tx + 4) (halo included), the wider on a tie; rows
// ty = tm_rows(tx); the maps start at the slab's first in-grid storage plane (planes outside the
// global grid read zeros).
int tm_tile_width(int ldx) {
  int best = TM_MAXTX, cost = INT_MAX;
  for (int tx = TM_MAXTX; tx >= 32; tx /= 2) {
    const int ntx = (ldx + 1 + tx - 1) / tx;
    if (ntx * (tx + 4) < cost) { cost = ntx * (tx + 4); best = tx; }
  }
  return best;
}
void tm_geometry(hz_coeffs* c) {
  const hz_grid& g = c->grid;
  const int tx = tm_tile_width(c->ldx);
  c->tm_tx = tx;
  c->tm_ty = tm_rows(tx);
  c->tm_org = g.z0 == 0 ? 1 : 0;
  const int last = (g.z0 + g.nz_local == g.nz_global) ? g.nz_local : g.nz_local + 1;
  c->tm_nval = last - c->tm_org + 1;
}

// 3-D (w: x, y, plane) or 4-D (u: x, y, plane, RHS) map of a pitched slab array; box = one halo tile
hz_status tm_encode(const hz_coeffs* c, CUtensorMap* map, const void* base, size_t esz, int nrhs) {
  HZ_TRY(tm_encoder());
  const hz_grid& g = c->grid;
  const char* org = reinterpret_cast<const char*>(base) + (size_t)c->tm_org * (size_t)c->plane() * esz;
  const cuuint64_t dims[4] = {(cuuint64_t)g.nx, (cuuint64_t)g.ny, (cuuint64_t)c->tm_nval, (cuuint64_t)nrhs};
  const cuuint64_t strides[3] = {(cuuint64_t)c->ldx * esz, (cuuint64_t)c->plane() * esz, (cuuint64_t)c->fstride() * esz};
  const cuuint32_t box[4] = {(cuuint32_t)(esz == 4 ? tm_bxw(c->tm_tx) : tm_bxu(c->tm_tx)), (cuuint32_t)(c->tm_ty + 2), 1u, 1u};
  const cuuint32_t estr[4] = {1u, 1u, 1u, 1u};
  const int rank = esz == 4 ? 3 : 4;
  CUresult r = g_encode(map, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank,
                        const_cast<char*>(org), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return HZ_ERR_CUDA;
  }
  return HZ_OK;
}

const CUtensorMap* tm_umap(hz_coeffs* c, const void* u, int nrhs) {
  const auto key = std::make_pair(u, nrhs);
  auto it = c->tmap_u.find(key);
  if (it != c->tmap_u.end()) return &it->second;
  if (c->tmap_u.size() >= 32) c->tmap_u.clear();
  CUtensorMap m;
  if (tm_encode(c, &m, u, 8, nrhs) != HZ_OK) return nullptr;
  return &(c->tmap_u[key] = m);
}

// Work list: the ntx × nty tiles, each marching the slab in z-chunks; every item runs once per RHS,
// handed out dynamically in list order.  A chunk re-reads 2 halo planes, and the schedule's makespan
// depends on how the items pack onto the CTAs, so the planner simulates the greedy list schedule
// (each item to the CTA that frees first; cost = planes read, x/y-PML tiles weighted 1.3) for n equal
// chunks per tile and for one long + one short chunk per tile (short ones last), and keeps the split
// with the shortest makespan.  Items of tiles holding x/y-PML points come first within a chunk;
// TM_PMLZ marks chunks holding z-PML output planes (the kernel tests each plane).  Chunk-major order:
// concurrently running CTAs work on neighbouring tiles at similar depths (halo rows shared in L2).
// the tiles of a plane: those holding x/y-PML points (xy) and the others (in)
void tm_tiles(const hz_grid& g, int ldx, int tx, int ty, const int lo[3], const int hi[3],
              std::vector<std::pair<int, int>>& xy, std::vector<std::pair<int, int>>& in) {
  const int ntx = (ldx + 1 + tx - 1) / tx, nty = (g.ny + ty - 1) / ty;
  for (int j = 0; j < nty; j++)
    for (int i = 0; i < ntx; i++) {
      const int x0 = i * tx, y0 = j * ty;   // computes columns [x0 − 1, x0 + tx − 1)
      const int xa = std::max(x0 - 1, 0), x1 = std::min(x0 + tx - 1, g.nx) - 1, y1 = std::min(y0 + ty, g.ny) - 1;
      const bool pml = xa < lo[0] || x1 > hi[0] || y0 < lo[1] || y1 > hi[1] || hi[0] < lo[0] || hi[1] < lo[1];
      (pml ? xy : in).push_back({x0, y0});
    }
}
// TM_PMLZ if the local output planes [a, b) of the slab hold z-PML planes
int tm_zmode(const hz_grid& g, const int lo[3], const int hi[3], int a, int b) {
  const int nzl = g.nz_local;
  const int zl = std::min(std::max(lo[2] - g.z0, 0), nzl);
  const int zh = std::min(std::max(hi[2] - g.z0 + 1, zl), nzl);
  return (a < zl || b > zh) ? TM_PMLZ : 0;
}
void tm_build_items(const hz_grid& g, int ldx, int tx, int ty, const int lo[3], const int hi[3], int slots, int nrhs,
                    std::vector<int4>& out) {
  const int nzl = g.nz_local;
  std::vector<std::pair<int, int>> xy, in;
  tm_tiles(g, ldx, tx, ty, lo, hi, xy, in);
  const int rep = std::max(1, nrhs);
  const int ncta = std::max(1, slots);
  auto makespan = [&](const std::vector<int>& cuts) {
    std::priority_queue<double, std::vector<double>, std::greater<double>> q;
    for (int k = 0; k < ncta; k++) q.push(0.0);
    double mk = 0.0;
    for (size_t k = 0; k + 1 < cuts.size(); k++) {
      const double L = cuts[k + 1] - cuts[k] + 2.0;
      for (int pass = 0; pass < 2; pass++) {
        const size_t cnt = (pass == 0 ? xy.size() : in.size()) * rep;
        const double cost = pass == 0 ? 1.3 * L : L;
        for (size_t i = 0; i < cnt; i++) {
          const double t = q.top() + cost;
          q.pop();
          q.push(t);
          mk = std::max(mk, t);
        }
      }
    }
    return mk;
  };
  std::vector<int> best_cuts{0, nzl};
  double best = makespan(best_cuts);
  for (int n = 2; n <= std::max(1, nzl / 3); n++) {
    std::vector<int> cuts;
    for (int k = 0; k <= n; k++) cuts.push_back((int)((long long)nzl * k / n));
    const double m = makespan(cuts);
    if (m < best - 1e-9) { best = m; best_cuts = cuts; }
  }
  for (int t = 2; t <= nzl / 2; t++) {
    const std::vector<int> cuts{0, nzl - t, nzl};
    const double m = makespan(cuts);
    if (m < best - 1e-9) { best = m; best_cuts = cuts; }
  }
  out.clear();
  for (size_t k = 0; k + 1 < best_cuts.size(); k++) {
    const int a = best_cuts[k], b = best_cuts[k + 1];
    const int zm = tm_zmode(g, lo, hi, a, b);
    for (auto& t : xy) out.push_back(tm_item(t.first, t.second, a, b, TM_PMLXY | zm));
    for (auto& t : in) out.push_back(tm_item(t.first, t.second, a, b, zm));
  }
}

const hz_coeffs::TmPlan* tm_plan(hz_coeffs* c, int nrhs) {
  auto it = c->tm_plans.find(nrhs);
  if (it != c->tm_plans.end()) return it->second.get();
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->ctx->device);
  std::vector<int4> items;
  // several slabs: the output planes next to an exchanged halo (local 0 below a lower neighbour,
  // nzl − 1 below an upper one) become one-plane items at the end of the list, so that the items
  // before them can run while the halo planes move (apply_launch)
  const hz_grid& g = c->grid;
  const int ia = (c->ctx->nranks > 1 && c->ctx->rank > 0) ? 1 : 0;
  const int ib = g.nz_local - ((c->ctx->nranks > 1 && c->ctx->rank < c->ctx->nranks - 1) ? 1 : 0);
  int n_int;
  if (c->ctx->nranks > 1 && ib - ia >= 2) {
    hz_grid gi = g;   // the interior planes [ia, ib) as a slab of their own
    gi.z0 += ia;
    gi.nz_local = ib - ia;
    tm_build_items(gi, c->ldx, c->tm_tx, c->tm_ty, c->lo, c->hi, sms, nrhs, items);
    for (int4& t : items) {
      const int a = (t.y & 0xffff) + ia, b = (t.y >> 16) + ia;
      t.y = a | (b << 16);
    }
    n_int = (int)items.size();
    std::vector<std::pair<int, int>> xy, in;
    tm_tiles(g, c->ldx, c->tm_tx, c->tm_ty, c->lo, c->hi, xy, in);
    for (int z : {0, g.nz_local - 1}) {
      if ((z == 0 && ia == 0) || (z == g.nz_local - 1 && ib == g.nz_local)) continue;
      const int zm = tm_zmode(g, c->lo, c->hi, z, z + 1);
      for (auto& t : xy) items.push_back(tm_item(t.first, t.second, z, z + 1, TM_PMLXY | zm));
      for (auto& t : in) items.push_back(tm_item(t.first, t.second, z, z + 1, zm));
    }
  } else {
    tm_build_items(g, c->ldx, c->tm_tx, c->tm_ty, c->lo, c->hi, sms, nrhs, items);
    n_int = c->ctx->nranks > 1 ? 0 : (int)items.size();   // thin slab: everything after the exchange
  }
  std::unique_ptr<hz_coeffs::TmPlan> pl(new hz_coeffs::TmPlan);
  pl->n_items = (int)items.size();
  pl->n_int = n_int;
  pl->grid = sms;   // one persistent CTA per SM
  if (pl->work.ensure(std::max<size_t>(1, items.size()) * sizeof(int4)) != cudaSuccess) return nullptr;
  if (!items.empty() && cudaMemcpy(pl->work.p, items.data(), items.size() * sizeof(int4), cudaMemcpyHostToDevice) != cudaSuccess)
    return nullptr;
  auto* raw = pl.get();
  c->tm_plans[nrhs] = std::move(pl);
  return raw;
}

}  // namespace

// test hook (include/hz_debug.h): the tensor-map apply's work list for a single slab
extern "C" int hz_debug_plan_tiles(int nx, int ny, int nz, int lo_x, int hi_x, int lo_y, int hi_y, int lo_z, int hi_z,
                                   int slots, int nrhs, int* out, int max_items, int* tile_wh) {
  if (nx < 3 || ny < 3 || nz < 1 || nx > 65535 || ny > 65535 || nz > 65535 || slots < 1 || nrhs < 1 ||
      (max_items > 0 && out == nullptr))
    return -1;
  hz_grid g{nx, ny, nz, 0, nz, 1.0, 0};
  const int ldx = hz_field_ldx(nx);
  const int tx = tm_tile_width(ldx);
  const int ty = tm_rows(tx);
  const int lo[3] = {lo_x, lo_y, lo_z}, hi[3] = {hi_x, hi_y, hi_z};
  std::vector<int4> items;
  tm_build_items(g, ldx, tx, ty, lo, hi, slots, nrhs, items);
  for (int n = 0; n < (int)items.size() && n < max_items; n++) {
    const int4 t = items[n];
    int* o = out + 5 * n;
    o[0] = t.x & 0xffff; o[1] = t.x >> 16; o[2] = t.y & 0xffff; o[3] = t.y >> 16; o[4] = t.z;
  }
  if (tile_wh) { tile_wh[0] = tx; tile_wh[1] = ty; }
  return (int)items.size();
}

namespace {

// One operator apply: complex64 (arithmetic and storage) through the tensor-map kernel, everything
// else (complex128, the fp64 residual of the complex64 solver) through the register path.  Dot
// epilogues get their partial / ticket scratch here.
// exch: first exchange the halo planes of p.u with the z neighbours (nranks > 1).  The complex64
// tensor-map apply overlaps that exchange with its interior items: they run on s while the halo
// planes move on the overlap stream, then the one-plane boundary items (and the dot reduction over
// the whole list) run after the join.  Every point is computed by the same operation sequence either
// way, so the output is bitwise that of the exchange-then-apply order.
template <typename R, typename S>
hz_status apply_launch(const hz_coeffs* cc, ApplyParams<R, S>& p, int nrhs, int epi, cudaStream_t s, bool exch = false) {
  hz_coeffs* c = const_cast<hz_coeffs*>(cc);
  typedef typename Cx<S>::T CU;
  const int K = epi_k(epi);
  constexpr bool TM = sizeof(R) == 4 && sizeof(S) == 4;
  const bool ovl = TM && exch && !c->medium && c->ctx->nranks > 1;
  if (exch && !ovl) HZ_TRY(halo_exchange(c, const_cast<CU*>(p.u), nrhs, sizeof(CU), s));
  if (c->medium) {   // visco-acoustic / variable density: the b-weighted gather kernel (apply_medium.cu)
    typedef typename Cx<S>::T CS;
    const S* bm = c->bmed.template as<S>();
    const CS* ki = c->kinv.template as<CS>();
    const bool colloc = c->mass == HZ_MASS_COLLOC;
    const long long nb = launch_apply_medium<R, S>(p, bm, ki, nrhs, colloc, epi, s, nullptr);
    if (K > 0) {
      HZ_CUDA(c->partials.ensure(sizeof(double) * (size_t)nb * K * nrhs));
      if (c->tickets.n < sizeof(unsigned) * (size_t)nrhs) {
        HZ_CUDA(c->tickets.ensure(sizeof(unsigned) * (size_t)nrhs));
        HZ_CUDA(cudaMemsetAsync(c->tickets.p, 0, c->tickets.n, s));
      }
      p.partials = c->partials.as<double>();
      p.tickets = c->tickets.as<unsigned>();
    }
    cudaError_t e = cudaSuccess;
    launch_apply_medium<R, S>(p, bm, ki, nrhs, colloc, epi, s, &e);
    HZ_CUDA(e);
    count_launch();
    return HZ_OK;
  }
  TmLaunch L{nullptr, nullptr, nullptr};
  CUtensorMap map_u, map_r;   // copies: a later tm_umap call may evict the cached entries
  const hz_coeffs::TmPlan* pl = nullptr;
  long long nb = 0;
  if constexpr (TM) {
    pl = tm_plan(c, nrhs);
    if (!pl) { set_error("tm_plan: device allocation / copy failed"); return HZ_ERR_CUDA; }
    if (c->tm_ctr.n == 0) {   // work counter + finished-CTA ticket, zero between launches
      HZ_CUDA(c->tm_ctr.ensure(2 * sizeof(unsigned)));
      HZ_CUDA(cudaMemsetAsync(c->tm_ctr.p, 0, 2 * sizeof(unsigned), s));
    }
    p.tm_work = pl->work.template as<int4>();
    p.tm_ctr = c->tm_ctr.template as<unsigned>();
    p.tm_item0 = 0;
    p.tm_nitems = pl->n_items;
    p.tm_nred = pl->n_items;
    p.tm_nblocks = std::max(1, std::min(pl->n_items * nrhs, pl->grid));   // persistent CTAs
    L.w = &c->tmap_w;
    const CUtensorMap* mu = tm_umap(c, p.u, nrhs);
    if (!mu) return HZ_ERR_CUDA;
    map_u = *mu;
    L.u = &map_u;
    if (K > 0) {   // the dot epilogues stage r̂₀ through TMA as well
      if (!p.rhat) { set_error("apply: dot epilogue without r-hat"); return HZ_ERR_INVALID_ARG; }
      const CUtensorMap* mr = tm_umap(c, p.rhat, nrhs);
      if (!mr) return HZ_ERR_CUDA;
      map_r = *mr;
      L.r = &map_r;
    }
    nb = (long long)pl->n_items;   // one dot partial slot per item and RHS
  } else {
    ApplyParams<R, S> pp = p;
    nb = apply_plan<R, S>(pp);
  }
  if (K > 0) {
    HZ_CUDA(c->partials.ensure(sizeof(double) * (size_t)nb * K * nrhs));
    if (c->tickets.n < sizeof(unsigned) * (size_t)nrhs) {
      HZ_CUDA(c->tickets.ensure(sizeof(unsigned) * (size_t)nrhs));
      HZ_CUDA(cudaMemsetAsync(c->tickets.p, 0, c->tickets.n, s));
    }
    p.partials = c->partials.as<double>();
    p.tickets = c->tickets.as<unsigned>();
  }
  if constexpr (TM) {
    const bool colloc = c->mass == HZ_MASS_COLLOC;
    if (ovl) {
      HZ_CUDA(c->ovl.init());
      HZ_CUDA(cudaEventRecord(c->ovl.fork, s));
      if (pl->n_int > 0) {   // interior items: no halo plane read
        ApplyParams<R, S> pi = p;
        pi.tm_nitems = pl->n_int;
        pi.tm_nred = 0;
        // NCCL moves the planes with its own kernels: leave them a few SMs (the loopback group copies
        // with the copy engines)
        const int spare = c->ctx->loop ? 0 : 4;
        pi.tm_nblocks = std::max(1, std::min(pl->n_int * nrhs, pl->grid - spare));
        HZ_CUDA(launch_apply_tm(L, pi, nrhs, colloc, epi, s));
        count_launch(apply_last_launches());
      }
      HZ_CUDA(cudaStreamWaitEvent(c->ovl.cs, c->ovl.fork, 0));
      HZ_TRY(halo_exchange(c, const_cast<CU*>(p.u), nrhs, sizeof(CU), c->ovl.cs));
      HZ_CUDA(cudaEventRecord(c->ovl.join, c->ovl.cs));
      HZ_CUDA(cudaStreamWaitEvent(s, c->ovl.join, 0));
      p.tm_item0 = pl->n_int;
      p.tm_nitems = pl->n_items - pl->n_int;
      p.tm_nblocks = std::max(1, std::min(p.tm_nitems * nrhs, pl->grid));
      if (p.tm_nitems == 0) return HZ_OK;
    }
    HZ_CUDA(launch_apply_tm(L, p, nrhs, colloc, epi, s));
  } else {
    HZ_CUDA(launch_apply<R, S>(p, nrhs, c->mass == HZ_MASS_COLLOC, epi, s));
  }
  count_launch(apply_last_launches());
  return HZ_OK;
}

template <typename R>
hz_status assemble_t(hz_ctx* ctx, const hz_grid* g, const void* v_in, double freq, const hz_pml* pml,
                     const hz_table* table, hz_mass mass, hz_rule rule, hz_coeffs** out, long long* n_clamped) {
  typedef typename Cx<R>::T C;
  std::unique_ptr<hz_coeffs> c(new hz_coeffs);
  c->ctx = ctx;
  c->dtype = sizeof(R) == 4 ? HZ_C64 : HZ_C128;
  c->grid = *g;
  c->mass = mass;
  c->rule = rule;
  c->freq = freq;
  c->omega = 2.0 * M_PI * freq;
  c->h = g->h;
  c->pml = pml ? *pml : hz_pml{0, 1e-3, 0.0};
  if (c->pml.npml < 0 || !(c->pml.r_coeff > 0) || c->pml.r_coeff > 1.0) {
    set_error("hz_assemble_coeffs: need npml >= 0 and 0 < r_coeff <= 1");
    return HZ_ERR_INVALID_ARG;
  }
  cudaStream_t s = 0;
  c->ldx = hz_field_ldx(g->nx);
  const long long plane = c->plane();
  const long long nloc = (long long)g->nx * g->ny * g->nz_local;   // owned points
  // ---- table: rank 0's rows broadcast to all ranks (bitwise-identical weights everywhere)
  c->table = table->t;
  if (ctx->nranks > 1) {
    DBuf tb;
    const size_t nb = 5 * (size_t)c->table.n_g * sizeof(double);
    HZ_CUDA(tb.ensure(nb));
    HZ_CUDA(cudaMemcpy(tb.p, c->table.rows5.data(), nb, cudaMemcpyHostToDevice));
    HZ_TRY(comm_bcast(ctx, tb.as<double>(), 5 * (size_t)c->table.n_g, s));
    HZ_CUDA(cudaMemcpy(c->table.rows5.data(), tb.p, nb, cudaMemcpyDeviceToHost));
  }
  // device table rows: (t1, t2, mu0, mu1, mu2 | forward differences), t1 = ws2/12, t2 = ws3/8 (A6)
  {
    const Table& T = c->table;
    const int ng = T.n_g < 2 ? 2 : T.n_g;
    std::vector<double> u(5 * (size_t)ng);
    for (int i = 0; i < ng; i++) {
      const double* w = &T.rows5[5 * (size_t)(T.n_g < 2 ? 0 : i)];
      u[5 * i + 0] = w[1] / 12.0;
      u[5 * i + 1] = (1.0 - w[0] - w[1]) / 8.0;
      u[5 * i + 2] = w[2];
      u[5 * i + 3] = w[3];
      u[5 * i + 4] = w[4];
    }
    std::vector<double> rows((size_t)ng * TAB_STRIDE, 0.0);
    for (int i = 0; i < ng; i++)
      for (int k = 0; k < 5; k++) {
        rows[(size_t)i * TAB_STRIDE + k] = u[5 * i + k];
        rows[(size_t)i * TAB_STRIDE + 5 + k] = (i + 1 < ng) ? (u[5 * (i + 1) + k] - u[5 * i + k]) : 0.0;
      }
    std::vector<float> rows_f(rows.size());
    for (size_t i = 0; i < rows.size(); i++) rows_f[i] = (float)rows[i];
    // apply table: class stiffness coefficients ×h⁻² (A6: centre −6t0, face t0−4t1, edge 2t1−2t2,
    // corner 3t2; t0 = 1 − 4t1 − 4t2) and mass ω²μ0..ω²μ3 (μ3 = (1 − μ0 − 6μ1 − 12μ2)/8), with
    // forward differences for the in-kernel linear interpolation (A13)
    const double ih2d = 1.0 / (g->h * g->h), w2d = c->omega * c->omega;
    std::vector<double> cr((size_t)ng * CTAB_STRIDE, 0.0);
    std::vector<double> v6((size_t)ng * 6);
    for (int i = 0; i < ng; i++) {
      const double t1 = u[5 * i + 0], t2 = u[5 * i + 1], mu0 = u[5 * i + 2], mu1 = u[5 * i + 3], mu2 = u[5 * i + 4];
      const double t0 = 1.0 - 4.0 * t1 - 4.0 * t2;
      const double mu3 = (1.0 - mu0 - 6.0 * mu1 - 12.0 * mu2) / 8.0;
      double* o = &v6[(size_t)i * 6];
      o[0] = ih2d * (t0 - 4.0 * t1);        // face   c1
      o[1] = ih2d * (2.0 * t1 - 2.0 * t2);  // edge   c2
      o[2] = ih2d * (3.0 * t2);             // corner c3   (centre c0 = −(6c1 + 12c2 + 8c3))
      o[3] = w2d * mu1;                     // m1 .. m3    (m0 = ω² − 6m1 − 12m2 − 8m3)
      o[4] = w2d * mu2;
      o[5] = w2d * mu3;
    }
    for (int i = 0; i < ng; i++) {
      double* o = &cr[(size_t)i * CTAB_STRIDE];
      for (int k = 0; k < 6; k++) {
        o[k] = v6[(size_t)i * 6 + k];
        o[6 + k] = (i + 1 < ng) ? v6[(size_t)(i + 1) * 6 + k] - v6[(size_t)i * 6 + k] : 0.0;
      }
    }
    std::vector<float> cr_f(cr.size());
    for (size_t i = 0; i < cr.size(); i++) cr_f[i] = (float)cr[i];
    // complex64 tensor-map apply: the centre coefficients tabulated too (c0 = −(6c1 + 12c2 + 8c3),
    // m0 = ω² − 6m1 − 12m2 − 8m3, evaluated in fp64), rows of TMTAB_STRIDE floats
    // [c0 c1 c2 c3 | m0 m1 m2 m3 | differences of the same eight]
    std::vector<float> ct_f((size_t)ng * TMTAB_STRIDE, 0.f);
    {
      std::vector<double> v8((size_t)ng * 8);
      for (int i = 0; i < ng; i++) {
        const double* o = &v6[(size_t)i * 6];
        double* q = &v8[(size_t)i * 8];
        q[0] = -(6.0 * o[0] + 12.0 * o[1] + 8.0 * o[2]);
        q[1] = o[0];
        q[2] = o[1];
        q[3] = o[2];
        q[4] = w2d - (6.0 * o[3] + 12.0 * o[4] + 8.0 * o[5]);
        q[5] = o[3];
        q[6] = o[4];
        q[7] = o[5];
      }
      for (int i = 0; i < ng; i++)
        for (int k = 0; k < 8; k++) {
          ct_f[(size_t)i * TMTAB_STRIDE + k] = (float)v8[(size_t)i * 8 + k];
          ct_f[(size_t)i * TMTAB_STRIDE + 8 + k] = (i + 1 < ng) ? (float)(v8[(size_t)(i + 1) * 8 + k] - v8[(size_t)i * 8 + k]) : 0.f;
        }
    }
    HZ_CUDA(c->ctab_d.ensure(cr.size() * sizeof(double)));
    HZ_CUDA(cudaMemcpy(c->ctab_d.p, cr.data(), cr.size() * sizeof(double), cudaMemcpyHostToDevice));
    if (sizeof(R) == 4) {
      HZ_CUDA(c->ctab_f.ensure(cr_f.size() * sizeof(float)));
      HZ_CUDA(cudaMemcpy(c->ctab_f.p, cr_f.data(), cr_f.size() * sizeof(float), cudaMemcpyHostToDevice));
      HZ_CUDA(c->ctm_f.ensure(ct_f.size() * sizeof(float)));
      HZ_CUDA(cudaMemcpy(c->ctm_f.p, ct_f.data(), ct_f.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
    c->n_g_dev = ng;
    c->g_min = T.g_min;
    c->dg = T.dg;
    c->g_max = T.n_g < 2 ? T.g_min + T.dg : T.g_min + T.dg * (T.n_g - 1);
    if ((size_t)ng * TAB_STRIDE * sizeof(R) > 60 * 1024) {
      set_error("hz_assemble_coeffs: table too large for shared memory");
      return HZ_ERR_INVALID_ARG;
    }
    HZ_CUDA(c->tab_d.ensure(rows.size() * sizeof(double)));
    HZ_CUDA(cudaMemcpy(c->tab_d.p, rows.data(), rows.size() * sizeof(double), cudaMemcpyHostToDevice));
    if (sizeof(R) == 4) {
      HZ_CUDA(c->tab_f.ensure(rows_f.size() * sizeof(float)));
      HZ_CUDA(cudaMemcpy(c->tab_f.p, rows_f.data(), rows_f.size() * sizeof(float), cudaMemcpyHostToDevice));
    }
  }
  // ---- velocity with halo planes
  // pitched [nzl+2][ny][ldx] copy of the caller's [nz][ny][nx] model; pad columns and the halo planes
  // outside the global grid stay 0 (never read as model values: the apply zero-fills those points)
  HZ_CUDA(c->v.ensure((size_t)(g->nz_local + 2) * plane * sizeof(R)));
  HZ_CUDA(cudaMemsetAsync(c->v.p, 0, (size_t)(g->nz_local + 2) * plane * sizeof(R), s));
  {
    const cudaMemcpyKind kind = is_device_ptr(v_in) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const R* vin = reinterpret_cast<const R*>(v_in);
    const size_t rowb = (size_t)g->nx * sizeof(R), pitch = (size_t)c->ldx * sizeof(R);
    const size_t vplane = (size_t)g->nx * g->ny;   // elements of one caller plane
    auto copy_planes = [&](int dst_plane, const R* src, int nplanes) {
      return cudaMemcpy2DAsync(c->v.as<R>() + (size_t)dst_plane * plane, pitch, src, rowb, rowb,
                               (size_t)nplanes * g->ny, kind, s);
    };
    if (g->v_halo) {
      HZ_CUDA(copy_planes(1, vin + vplane, g->nz_local));
      if (g->z0 > 0) HZ_CUDA(copy_planes(0, vin, 1));
      if (g->z0 + g->nz_local < g->nz_global) HZ_CUDA(copy_planes(g->nz_local + 1, vin + (size_t)(g->nz_local + 1) * vplane, 1));
    } else {
      HZ_CUDA(copy_planes(1, vin, g->nz_local));
    }
  }
  // ---- statistics: domain check, v range, clamps
  DBuf st;
  HZ_CUDA(st.ensure(4 * sizeof(unsigned long long)));
  unsigned long long init[4] = {~0ULL, 0ULL, 0ULL, 0ULL};
  HZ_CUDA(cudaMemcpy(st.p, init, sizeof(init), cudaMemcpyHostToDevice));
  HZ_CUDA(launch_vstats<R>(c->v.as<R>() + plane, nloc, g->nx, c->ldx, (R)(1.0 / (freq * g->h)), (R)c->g_min,
                           (R)c->g_max, st.as<unsigned long long>(), s));
  count_launch();
  unsigned long long res[4];
  HZ_CUDA(cudaMemcpy(res, st.p, sizeof(res), cudaMemcpyDeviceToHost));
  double vmin, vmax;
  {
    long long bmin = (long long)res[0], bmax = (long long)res[1];
    memcpy(&vmin, &bmin, 8);
    memcpy(&vmax, &bmax, 8);
  }
  double stats[3] = {(double)res[2], (double)res[3], 0.0};
  if (ctx->nranks > 1) {
    DBuf sb;
    HZ_CUDA(sb.ensure(4 * sizeof(double)));
    double sv[4] = {stats[0], stats[1], vmax, -vmin};
    HZ_CUDA(cudaMemcpy(sb.p, sv, sizeof(sv), cudaMemcpyHostToDevice));
    HZ_TRY(comm_allreduce(ctx, sb.as<double>(), 2, 0, s));
    HZ_TRY(comm_allreduce(ctx, sb.as<double>() + 2, 2, 1, s));
    HZ_CUDA(cudaMemcpy(sv, sb.p, sizeof(sv), cudaMemcpyDeviceToHost));
    stats[0] = sv[0];
    stats[1] = sv[1];
    vmax = sv[2];
    vmin = -sv[3];
  }
  if (stats[0] > 0) {
    set_error("hz_assemble_coeffs: velocity has " + std::to_string((long long)stats[0]) +
              " non-positive or non-finite values (S:156, S:252)");
    return HZ_ERR_DOMAIN;
  }
  // ---- v halo planes from the neighbours
  if (!g->v_halo) HZ_TRY(halo_exchange(c.get(), c->v.p, 1, sizeof(R), s));
  HZ_CUDA(c->w.ensure((size_t)(g->nz_local + 2) * plane * sizeof(R)));
  HZ_CUDA(launch_winv<R>(c->v.as<R>(), c->w.as<R>(), (long long)(g->nz_local + 2) * plane, s));
  count_launch();
  // ---- table rows the apply stages in shared memory: G range of the model (all ranks) ± 1 row
  {
    const double inv_fh = 1.0 / (freq * g->h);
    auto row_of = [&](double vv) {
      const double sidx = (vv * inv_fh - c->g_min) / c->dg;
      return (int)std::floor(std::fmin(std::fmax(sidx, 0.0), (double)(c->n_g_dev - 1)));
    };
    const int lo_r = std::max(0, std::min(row_of(vmin) - 1, c->n_g_dev - 2));
    const int hi_r = std::max(lo_r + 1, std::min(row_of(vmax) + 2, c->n_g_dev - 1));
    c->tab_lo = lo_r;
    c->tab_n = hi_r - lo_r + 1;
  }
  // ---- PML (host, double) → device deltas δ± = a± − 1/h²
  c->vmin = vmin;
  c->vmax = vmax;
  c->v_pml = (c->pml.v_pml > 0) ? c->pml.v_pml : vmax;
  const int ns[3] = {g->nx, g->ny, g->nz_global};
  const double ih2 = 1.0 / (g->h * g->h);
  for (int a = 0; a < 3; a++) {
    pml_axis(ns[a], c->pml.npml, g->h, c->omega, c->v_pml, c->pml.r_coeff, c->am_h[a], c->ap_h[a]);
    std::vector<float2> dm(ns[a]), dp(ns[a]);
    std::vector<double2> dmd(ns[a]), dpd(ns[a]);
    int lo = ns[a], hi = -1;
    for (int i = 0; i < ns[a]; i++) {
      std::complex<double> m = c->am_h[a][i] - ih2, q = c->ap_h[a][i] - ih2;
      dm[i].x = (float)m.real(); dm[i].y = (float)m.imag();
      dp[i].x = (float)q.real(); dp[i].y = (float)q.imag();
      dmd[i].x = m.real(); dmd[i].y = m.imag();
      dpd[i].x = q.real(); dpd[i].y = q.imag();
    }
    // interior range: the longest run of exactly-zero deltas (contiguous by construction)
    for (int i = 0; i < ns[a]; i++) {
      bool z = (c->am_h[a][i] - ih2) == std::complex<double>(0, 0) && (c->ap_h[a][i] - ih2) == std::complex<double>(0, 0);
      if (z) { if (i < lo) lo = i; hi = i; }
    }
    if (hi < lo) { lo = 1; hi = 0; }   // every node needs the correction
    c->lo[a] = lo;
    c->hi[a] = hi;
    HZ_CUDA(c->pml_d[a].ensure(ns[a] * sizeof(double2)));
    HZ_CUDA(c->pml_d[3 + a].ensure(ns[a] * sizeof(double2)));
    HZ_CUDA(cudaMemcpy(c->pml_d[a].p, dmd.data(), ns[a] * sizeof(double2), cudaMemcpyHostToDevice));
    HZ_CUDA(cudaMemcpy(c->pml_d[3 + a].p, dpd.data(), ns[a] * sizeof(double2), cudaMemcpyHostToDevice));
    if (sizeof(R) == 4) {
      HZ_CUDA(c->pml_f[a].ensure(ns[a] * sizeof(float2)));
      HZ_CUDA(c->pml_f[3 + a].ensure(ns[a] * sizeof(float2)));
      HZ_CUDA(cudaMemcpy(c->pml_f[a].p, dm.data(), ns[a] * sizeof(float2), cudaMemcpyHostToDevice));
      HZ_CUDA(cudaMemcpy(c->pml_f[3 + a].p, dp.data(), ns[a] * sizeof(float2), cudaMemcpyHostToDevice));
    }
  }
  // ---- launch geometry: strips of NY rows; z chunks sized to give >= ~4 waves
  {
    const long long bx = apply_nblocks_x<double>(g->nx, g->ny);
    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, ctx->device);
    const long long target = 4LL * dev_sms * apply_occupancy<double>(mass == HZ_MASS_COLLOC);
    long long nch = (target + bx - 1) / bx;
    const long long maxch = std::max(1, g->nz_local / 8);
    nch = std::max(1LL, std::min(nch, maxch));
    c->zc = (int)((g->nz_local + nch - 1) / nch);
    c->nchunks = (g->nz_local + c->zc - 1) / c->zc;
  }
  if (sizeof(R) == 4) {   // complex64: tile geometry and the tensor map of w for apply27_tm
    tm_geometry(c.get());
    HZ_TRY(tm_encode(c.get(), &c->tmap_w, c->w.p, 4, 1));
  }
  // ---- GAm: the 27-node mean weights of every owned row, once (A19)
  if (rule != HZ_RULE_GA) {
    HZ_CUDA(c->gam.ensure(5 * (size_t)c->fstride() * sizeof(R)));
    HZ_CUDA(cudaMemsetAsync(c->gam.p, 0, 5 * (size_t)c->fstride() * sizeof(R), s));
    ApplyParams<R> gp = make_params<R>(c.get());
    HZ_CUDA(launch_gam_field<R>(gp, c->gam.as<R>(), rule == HZ_RULE_GAM ? 1 : 0, s));
    count_launch();
    HZ_CUDA(cudaStreamSynchronize(s));
  }
  if (n_clamped) *n_clamped = (long long)stats[1];
  *out = c.release();
  return stats[1] > 0 ? HZ_WARN_CLAMPED : HZ_OK;
}

}  // namespace

extern "C" {

hz_status hz_assemble_coeffs(hz_ctx* ctx, const hz_grid* grid, hz_dtype dtype, const void* v, double freq_hz,
                             const hz_pml* pml, const hz_table* table, hz_mass mass, hz_rule rule, hz_coeffs** out,
                             long long* n_clamped) {
  if (!ctx || !grid || !v || !table || !out) { set_error("hz_assemble_coeffs: NULL argument"); return HZ_ERR_INVALID_ARG; }
  const hz_grid& g = *grid;
  if (g.nx < 3 || g.ny < 3 || g.nz_global < 3 || g.nz_local < 1 || g.z0 < 0 || g.z0 + g.nz_local > g.nz_global) {
    set_error("hz_assemble_coeffs: bad grid (dims >= 3, slab inside the global grid; S:156)");
    return HZ_ERR_INVALID_ARG;
  }
  if (g.nx > 65532 || g.ny > 65535 || g.nz_local > 65535) {
    set_error("hz_assemble_coeffs: nx <= 65532, ny and nz_local <= 65535 (apply work-item packing)");
    return HZ_ERR_INVALID_ARG;
  }
  if ((long long)(g.nz_local + 2) * hz_field_ldx(g.nx) * g.ny >= (1LL << 31)) {
    set_error("hz_assemble_coeffs: slab of >= 2^31 points per field (32-bit offsets in the apply); "
              "split the grid over more z-slabs");
    return HZ_ERR_INVALID_ARG;
  }
  if (!(g.h > 0) || !(freq_hz > 0)) { set_error("hz_assemble_coeffs: need h > 0 and f > 0 (S:172)"); return HZ_ERR_DOMAIN; }
  if (table->t.n_g < 1) { set_error("hz_assemble_coeffs: empty table"); return HZ_ERR_INVALID_ARG; }
  if (ctx->nranks > 1 && g.nz_local < 1) { set_error("hz_assemble_coeffs: empty slab"); return HZ_ERR_INVALID_ARG; }
  if (cudaSetDevice(ctx->device) != cudaSuccess) { set_error("hz_assemble_coeffs: cudaSetDevice failed"); return HZ_ERR_CUDA; }
  if (rule != HZ_RULE_GA && rule != HZ_RULE_GAM && rule != HZ_RULE_GA_RECORD) { set_error("hz_assemble_coeffs: bad rule"); return HZ_ERR_INVALID_ARG; }
  if (dtype == HZ_C64) return assemble_t<float>(ctx, grid, v, freq_hz, pml, table, mass, rule, out, n_clamped);
  if (dtype == HZ_C128) return assemble_t<double>(ctx, grid, v, freq_hz, pml, table, mass, rule, out, n_clamped);
  set_error("hz_assemble_coeffs: bad dtype");
  return HZ_ERR_INVALID_ARG;
}

void hz_coeffs_destroy(hz_coeffs* c) {
  if (!c) return;
  // buffers go back to the cache for reuse: let queued work that still reads them finish first
  cudaSetDevice(c->ctx->device);
  cudaDeviceSynchronize();
  delete c;
}

hz_status hz_coeffs_export(const hz_coeffs* c, void* record, void* pml_host, int nmax) {
  if (!c) { set_error("hz_coeffs_export: NULL coeffs"); return HZ_ERR_INVALID_ARG; }
  HZ_TRY(set_device(c->ctx));
  cudaStream_t s = 0;
  if (record) {
    const size_t nb = 8 * (size_t)c->npoints() * c->esz();
    const bool dev = is_device_ptr(record);
    DBuf tmp;
    void* dst = record;
    if (!dev) {
      HZ_CUDA(tmp.ensure(nb));
      dst = tmp.p;
    }
    if (c->dtype == HZ_C64) {
      auto p = make_params<float>(c);
      HZ_CUDA(launch_record<float>(p, reinterpret_cast<float*>(dst), s));
    } else {
      auto p = make_params<double>(c);
      HZ_CUDA(launch_record<double>(p, reinterpret_cast<double*>(dst), s));
    }
    count_launch();
    HZ_CUDA(cudaStreamSynchronize(s));
    if (!dev) HZ_CUDA(cudaMemcpy(record, tmp.p, nb, cudaMemcpyDeviceToHost));
  }
  if (pml_host) {
    const int ns[3] = {c->grid.nx, c->grid.ny, c->grid.nz_global};
    if (nmax < std::max(ns[0], std::max(ns[1], ns[2]))) { set_error("hz_coeffs_export: nmax too small"); return HZ_ERR_INVALID_ARG; }
    std::complex<double>* o = reinterpret_cast<std::complex<double>*>(pml_host);
    for (int a = 0; a < 3; a++)
      for (int i = 0; i < nmax; i++) {
        o[(size_t)(2 * a + 0) * nmax + i] = i < ns[a] ? c->am_h[a][i] : 0.0;
        o[(size_t)(2 * a + 1) * nmax + i] = i < ns[a] ? c->ap_h[a][i] : 0.0;
      }
  }
  return HZ_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------------
// (3) apply
// ---------------------------------------------------------------------------------------------
template <typename R>
static hz_status apply_t(const hz_coeffs* cc, void* u, void* au, int nrhs, cudaStream_t s) {
  typedef typename Cx<R>::T C;
  hz_coeffs* c = const_cast<hz_coeffs*>(cc);
  const size_t fsb = (size_t)c->fstride() * sizeof(C);   // bytes of one field
  const bool du = is_device_ptr(u), da = is_device_ptr(au);
  if (du && da) {
    ApplyParams<R> p = make_params<R>(c);
    p.u = reinterpret_cast<const C*>(u);
    p.au = reinterpret_cast<C*>(au);
    return apply_launch<R>(c, p, nrhs, EPI_PLAIN, s, true);
  }
  // host u and / or Au: RHS groups of g fields through two staging slots; group k's H2D copy (stream
  // in), apply (s) and D2H copy (stream out) overlap with the neighbouring groups'
  auto& io = c->hio;
  HZ_CUDA(io.init());
  const int g = std::min(nrhs, 2);
  if (!du) HZ_CUDA(io.bin.ensure(2 * g * fsb));
  if (!da) HZ_CUDA(io.bout.ensure(2 * g * fsb));
  HZ_CUDA(cudaEventRecord(io.start, s));   // the copies follow the caller's earlier work on s
  HZ_CUDA(cudaStreamWaitEvent(io.in, io.start, 0));
  HZ_CUDA(cudaStreamWaitEvent(io.out, io.start, 0));
  const int ng = (nrhs + g - 1) / g;
  for (int k = 0; k < ng; k++) {
    const int slot = k & 1, r0 = k * g, n = std::min(g, nrhs - r0);
    const size_t off = (size_t)r0 * fsb, bytes = (size_t)n * fsb;
    char* src = du ? static_cast<char*>(u) + off : io.bin.as<char>() + (size_t)slot * g * fsb;
    char* dst = da ? static_cast<char*>(au) + off : io.bout.as<char>() + (size_t)slot * g * fsb;
    if (!du) {
      if (k >= 2) HZ_CUDA(cudaStreamWaitEvent(io.in, io.e_comp[slot], 0));   // group k-2 has read the slot
      HZ_CUDA(cudaMemcpyAsync(src, static_cast<const char*>(u) + off, bytes, cudaMemcpyHostToDevice, io.in));
      HZ_CUDA(cudaEventRecord(io.e_in[slot], io.in));
      HZ_CUDA(cudaStreamWaitEvent(s, io.e_in[slot], 0));
    }
    if (!da && k >= 2) HZ_CUDA(cudaStreamWaitEvent(s, io.e_out[slot], 0));   // group k-2's result copied out
    ApplyParams<R> p = make_params<R>(c);
    p.u = reinterpret_cast<const C*>(src);
    p.au = reinterpret_cast<C*>(dst);
    HZ_TRY(apply_launch<R>(c, p, n, EPI_PLAIN, s, true));
    HZ_CUDA(cudaEventRecord(io.e_comp[slot], s));
    if (!da) {
      HZ_CUDA(cudaStreamWaitEvent(io.out, io.e_comp[slot], 0));
      HZ_CUDA(cudaMemcpyAsync(static_cast<char*>(au) + off, dst, bytes, cudaMemcpyDeviceToHost, io.out));
      HZ_CUDA(cudaEventRecord(io.e_out[slot], io.out));
    }
  }
  if (!da)
    for (int k = 0; k < std::min(ng, 2); k++) HZ_CUDA(cudaStreamWaitEvent(s, io.e_out[k], 0));
  HZ_CUDA(cudaStreamSynchronize(s));
  return HZ_OK;
}

template <typename R>
static hz_status set_medium_t(hz_coeffs* c, const void* b, const void* q, cudaStream_t s) {
  const hz_grid* g = &c->grid;
  const long long plane = c->plane(), n = (long long)(g->nz_local + 2) * plane;
  DBuf qd;
  auto load = [&](DBuf& dst, const void* src, R fill) -> hz_status {
    HZ_CUDA(dst.ensure((size_t)n * sizeof(R)));
    HZ_CUDA(launch_medium_fill<R>(dst.as<R>(), n, fill, s));
    count_launch();
    if (src == nullptr) return HZ_OK;
    const cudaMemcpyKind kind = is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    const R* in = reinterpret_cast<const R*>(src);
    const size_t rowb = (size_t)g->nx * sizeof(R), pitch = (size_t)c->ldx * sizeof(R);
    const size_t vplane = (size_t)g->nx * g->ny;
    auto copy_planes = [&](int dst_plane, const R* sp, int np) {
      return cudaMemcpy2DAsync(dst.as<R>() + (size_t)dst_plane * plane, pitch, sp, rowb, rowb, (size_t)np * g->ny, kind, s);
    };
    if (g->v_halo) {   // the same layout as v (include/hz.h hz_grid.v_halo)
      HZ_CUDA(copy_planes(1, in + vplane, g->nz_local));
      if (g->z0 > 0) HZ_CUDA(copy_planes(0, in, 1));
      if (g->z0 + g->nz_local < g->nz_global) HZ_CUDA(copy_planes(g->nz_local + 1, in + (size_t)(g->nz_local + 1) * vplane, 1));
    } else {
      HZ_CUDA(copy_planes(1, in, g->nz_local));
      HZ_TRY(halo_exchange(c, dst.p, 1, sizeof(R), s));
    }
    return HZ_OK;
  };
  HZ_TRY(load(c->bmed, b, R(1)));
  if (q) HZ_TRY(load(qd, q, R(0)));
  DBuf bad;
  HZ_CUDA(bad.ensure(sizeof(unsigned long long)));
  HZ_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(unsigned long long), s));
  HZ_CUDA(launch_medium_check<R>(c->bmed.as<R>() + plane, q ? qd.as<R>() + plane : nullptr, (long long)g->nz_local * plane,
                                 g->nx, c->ldx, bad.as<unsigned long long>(), s));
  count_launch();
  unsigned long long nbad = 0;
  HZ_CUDA(cudaMemcpyAsync(&nbad, bad.p, sizeof(nbad), cudaMemcpyDeviceToHost, s));
  HZ_CUDA(cudaStreamSynchronize(s));
  if (nbad > 0) {
    set_error("hz_coeffs_set_medium: " + std::to_string(nbad) + " buoyancy / Q values are not positive and finite");
    return HZ_ERR_DOMAIN;
  }
  typedef typename Cx<R>::T C;
  HZ_CUDA(c->kinv.ensure((size_t)n * sizeof(C)));
  HZ_CUDA(launch_medium_kinv<R>(c->v.as<R>(), c->bmed.as<R>(), q ? qd.as<R>() : nullptr, c->kinv.as<C>(), n, s));
  count_launch();
  HZ_CUDA(cudaStreamSynchronize(s));
  c->medium = true;
  return HZ_OK;
}

extern "C" hz_status hz_coeffs_set_medium(hz_coeffs* c, const void* b, const void* q, void* stream) {
  if (!c) { set_error("hz_coeffs_set_medium: NULL coeffs"); return HZ_ERR_INVALID_ARG; }
  HZ_TRY(set_device(c->ctx));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (!b && !q) {   // ρ = 1, Q = ∞: back to the class-sum kernels
    c->medium = false;
    return HZ_OK;
  }
  return c->dtype == HZ_C64 ? set_medium_t<float>(c, b, q, s) : set_medium_t<double>(c, b, q, s);
}

extern "C" hz_status hz_apply_impedance(const hz_coeffs* c, void* u, void* au, int nrhs, void* stream) {
  if (!c || !u || !au || nrhs < 1) { set_error("hz_apply_impedance: bad arguments"); return HZ_ERR_INVALID_ARG; }
  if (u == au) { set_error("hz_apply_impedance: u and au must not alias"); return HZ_ERR_INVALID_ARG; }
  HZ_TRY(set_device(c->ctx));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return c->dtype == HZ_C64 ? apply_t<float>(c, u, au, nrhs, s) : apply_t<double>(c, u, au, nrhs, s);
}

// ---------------------------------------------------------------------------------------------
// point sources
// ---------------------------------------------------------------------------------------------
template <typename R>
static hz_status sources_t(const hz_coeffs* c, int nsrc, const long long* nodes, const double* amps, int consistent,
                           void* b, cudaStream_t s) {
  typedef typename Cx<R>::T C;
  const int np = c->pml.npml;
  for (int i = 0; i < nsrc; i++) {
    const long long X = nodes[3 * i], Y = nodes[3 * i + 1], Z = nodes[3 * i + 2];
    if (X < 0 || X >= c->grid.nx || Y < 0 || Y >= c->grid.ny || Z < 0 || Z >= c->grid.nz_global) {
      set_error("hz_point_sources: source outside the grid");
      return HZ_ERR_INVALID_ARG;
    }
    if (X < np || X >= c->grid.nx - np || Y < np || Y >= c->grid.ny - np || Z < np || Z >= c->grid.nz_global - np) {
      set_error("hz_point_sources: source " + std::to_string(i) + " lies inside the PML (S:262-266)");
      return HZ_ERR_SOURCE_IN_PML;
    }
  }
  const size_t fb = (size_t)c->fstride() * nsrc * sizeof(C);
  const bool db = is_device_ptr(b);
  DBuf tb, dn, da;
  void* bd = b;
  if (!db) { HZ_CUDA(tb.ensure(fb)); bd = tb.p; }
  HZ_CUDA(dn.ensure(3 * sizeof(long long) * nsrc));
  HZ_CUDA(cudaMemcpyAsync(dn.p, nodes, 3 * sizeof(long long) * nsrc, cudaMemcpyHostToDevice, s));
  if (amps) {
    HZ_CUDA(da.ensure(2 * sizeof(double) * nsrc));
    HZ_CUDA(cudaMemcpyAsync(da.p, amps, 2 * sizeof(double) * nsrc, cudaMemcpyHostToDevice, s));
  }
  HZ_CUDA(cudaMemsetAsync(bd, 0, fb, s));
  ApplyParams<R> p = make_params<R>(c);
  const R ih3 = (R)(1.0 / (c->h * c->h * c->h));
  HZ_CUDA(launch_sources<R>(p, nsrc, dn.as<long long>(), amps ? da.as<double>() : nullptr, consistent, ih3,
                            reinterpret_cast<C*>(bd), s));
  count_launch();
  if (!db) HZ_CUDA(cudaMemcpyAsync(b, bd, fb, cudaMemcpyDeviceToHost, s));
  HZ_CUDA(cudaStreamSynchronize(s));
  return HZ_OK;
}

extern "C" hz_status hz_point_sources(const hz_coeffs* c, int nsrc, const long long* node_xyz,
                                      const double* amp_re_im, int consistent, void* b, void* stream) {
  if (!c || nsrc < 1 || !node_xyz || !b) { set_error("hz_point_sources: bad arguments"); return HZ_ERR_INVALID_ARG; }
  HZ_TRY(set_device(c->ctx));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return c->dtype == HZ_C64 ? sources_t<float>(c, nsrc, node_xyz, amp_re_im, consistent, b, s)
                            : sources_t<double>(c, nsrc, node_xyz, amp_re_im, consistent, b, s);
}



// ---------------------------------------------------------------------------------------------
// evaluation: eqerror and the stencil's plane-wave dispersion
// ---------------------------------------------------------------------------------------------
template <typename R>
static hz_status eqerror_t(const hz_coeffs* c, const void* uref, const void* u, const long long* src, int npml,
                           double ball, double* err, cudaStream_t s) {
  typedef typename Cx<R>::T C;
  const size_t fb = (size_t)c->fstride() * sizeof(C);
  DBuf tr, tu, part;
  const void* rd = uref;
  const void* ud = u;
  if (!is_device_ptr(uref)) { HZ_CUDA(tr.ensure(fb)); HZ_CUDA(cudaMemcpyAsync(tr.p, uref, fb, cudaMemcpyHostToDevice, s)); rd = tr.p; }
  if (!is_device_ptr(u)) { HZ_CUDA(tu.ensure(fb)); HZ_CUDA(cudaMemcpyAsync(tu.p, u, fb, cudaMemcpyHostToDevice, s)); ud = tu.p; }
  const int nb = 148 * 4;
  HZ_CUDA(part.ensure(sizeof(double) * 4 * nb));
  const hz_grid& g = c->grid;
  HZ_CUDA(launch_eqerror<R>(reinterpret_cast<const C*>(rd), reinterpret_cast<const C*>(ud), g.nx, g.ny, c->ldx, g.nz_local,
                            g.z0, g.nz_global, src, g.h, npml, ball, part.as<double>(), nb, s));
  count_launch();
  std::vector<double> hp(4 * nb);
  HZ_CUDA(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * 4 * nb, cudaMemcpyDeviceToHost, s));
  HZ_CUDA(cudaStreamSynchronize(s));
  double sum[4] = {0, 0, 0, 0};
  for (int b = 0; b < nb; b++)
    for (int k = 0; k < 4; k++) sum[k] += hp[4 * b + k];
  if (c->ctx->nranks > 1) {
    DBuf d4;
    HZ_CUDA(d4.ensure(sizeof(sum)));
    HZ_CUDA(cudaMemcpyAsync(d4.p, sum, sizeof(sum), cudaMemcpyHostToDevice, s));
    HZ_TRY(allreduce_sum(c, d4.as<double>(), 4, s));
    HZ_CUDA(cudaMemcpyAsync(sum, d4.p, sizeof(sum), cudaMemcpyDeviceToHost, s));
    HZ_CUDA(cudaStreamSynchronize(s));
  }
  if (!(sum[2] > 0) || !(sum[3] > 0)) { set_error("hz_eqerror: degenerate reference field"); return HZ_ERR_DOMAIN; }
  *err = sum[0] / sum[2] + sum[1] / sum[3];
  return HZ_OK;
}

extern "C" hz_status hz_eqerror(const hz_coeffs* c, const void* u_ref, const void* u, const long long src_xyz[3],
                                int npml_mask, double ball_cells, double* err_out, void* stream) {
  if (!c || !u_ref || !u || !src_xyz || !err_out || npml_mask < 0) { set_error("hz_eqerror: bad arguments"); return HZ_ERR_INVALID_ARG; }
  HZ_TRY(set_device(c->ctx));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return c->dtype == HZ_C64 ? eqerror_t<float>(c, u_ref, u, src_xyz, npml_mask, ball_cells, err_out, s)
                            : eqerror_t<double>(c, u_ref, u, src_xyz, npml_mask, ball_cells, err_out, s);
}

template <typename R>
static hz_status matrix_t(const hz_coeffs* c, long long* cols, void* vals, cudaStream_t s) {
  typedef typename Cx<R>::T C;
  const size_t n = (size_t)c->npoints() * 27;
  DBuf dc, dv;
  long long* cd = cols;
  void* vd = vals;
  const bool cdev = is_device_ptr(cols), vdev = is_device_ptr(vals);
  if (!cdev) { HZ_CUDA(dc.ensure(n * sizeof(long long))); cd = dc.as<long long>(); }
  if (!vdev) { HZ_CUDA(dv.ensure(n * sizeof(C))); vd = dv.p; }
  ApplyParams<R> p = make_params<R>(c);
  HZ_CUDA(launch_matrix<R>(p, c->mass == HZ_MASS_COLLOC, cd, reinterpret_cast<C*>(vd), s));
  count_launch();
  if (!cdev) HZ_CUDA(cudaMemcpyAsync(cols, cd, n * sizeof(long long), cudaMemcpyDeviceToHost, s));
  if (!vdev) HZ_CUDA(cudaMemcpyAsync(vals, vd, n * sizeof(C), cudaMemcpyDeviceToHost, s));
  HZ_CUDA(cudaStreamSynchronize(s));
  return HZ_OK;
}

extern "C" hz_status hz_export_matrix(const hz_coeffs* c, long long* cols, void* vals, void* stream) {
  if (!c || !cols || !vals) { set_error("hz_export_matrix: bad arguments"); return HZ_ERR_INVALID_ARG; }
  HZ_TRY(set_device(c->ctx));
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return c->dtype == HZ_C64 ? matrix_t<float>(c, cols, vals, s) : matrix_t<double>(c, cols, vals, s);
}

extern "C" hz_status hz_table_dispersion(const hz_table* t, int nG, const double* G, int nang, const double* theta,
                                         const double* phi, double* vtilde, void* stream) {
  if (!t || nG < 1 || nang < 1 || !G || !theta || !phi || !vtilde) { set_error("hz_table_dispersion: bad arguments"); return HZ_ERR_INVALID_ARG; }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  // class weights at each G: clamped linear interpolation of the table's free weights (A13)
  const Table& T = t->t;
  std::vector<double> w7(7 * (size_t)nG), gv(G, G + nG);
  for (int i = 0; i < nG; i++) {
    if (!(G[i] > 0) || !std::isfinite(G[i])) { set_error("hz_table_dispersion: G must be finite and > 0"); return HZ_ERR_DOMAIN; }
    double u[5];
    if (T.n_g == 1) {
      for (int k = 0; k < 5; k++) u[k] = T.rows5[k];
    } else {
      const double gmax = T.g_min + T.dg * (T.n_g - 1);
      const double sidx = (std::fmin(std::fmax(G[i], T.g_min), gmax) - T.g_min) / T.dg;
      const int ii = std::min((int)std::floor(sidx), T.n_g - 2);
      const double tau = sidx - ii;
      for (int k = 0; k < 5; k++) u[k] = (1.0 - tau) * T.rows5[5 * ii + k] + tau * T.rows5[5 * (ii + 1) + k];
    }
    double* o = &w7[7 * (size_t)i];
    o[0] = u[0];
    o[1] = u[1];
    o[2] = 1.0 - u[0] - u[1];
    o[3] = u[2];
    o[4] = 6.0 * u[3];
    o[5] = 12.0 * u[4];
    o[6] = 1.0 - o[3] - o[4] - o[5];
  }
  DBuf dw, dg, dt, dp, dout;
  HZ_CUDA(dw.ensure(w7.size() * sizeof(double)));
  HZ_CUDA(dg.ensure(gv.size() * sizeof(double)));
  HZ_CUDA(dt.ensure(sizeof(double) * nang));
  HZ_CUDA(dp.ensure(sizeof(double) * nang));
  HZ_CUDA(dout.ensure(sizeof(double) * (size_t)nG * nang));
  HZ_CUDA(cudaMemcpyAsync(dw.p, w7.data(), w7.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  HZ_CUDA(cudaMemcpyAsync(dg.p, gv.data(), gv.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  HZ_CUDA(cudaMemcpyAsync(dt.p, theta, sizeof(double) * nang, cudaMemcpyHostToDevice, s));
  HZ_CUDA(cudaMemcpyAsync(dp.p, phi, sizeof(double) * nang, cudaMemcpyHostToDevice, s));
  HZ_CUDA(launch_dispersion(dw.as<double>(), dg.as<double>(), nG, dt.as<double>(), dp.as<double>(), nang, dout.as<double>(), s));
  count_launch();
  HZ_CUDA(cudaMemcpyAsync(vtilde, dout.p, sizeof(double) * (size_t)nG * nang, cudaMemcpyDefault, s));
  HZ_CUDA(cudaStreamSynchronize(s));
  return HZ_OK;
}

// ---------------------------------------------------------------------------------------------
// (4) batched BiCGSTAB (north star (3); reading A21)
// ---------------------------------------------------------------------------------------------
namespace {

struct EventTimer {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  size_t used = 0;
  ~EventTimer() { for (auto e : ev) cudaEventDestroy(e); }
  void mark(cudaStream_t s) {
    if (!on) return;
    if (used == ev.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev.push_back(e);
    }
    cudaEventRecord(ev[used++], s);
  }
  double total_ms() {
    double t = 0;
    for (size_t i = 0; i + 1 < used; i += 2) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      t += ms;
    }
    return t;
  }
};

template <typename R>
hz_status solve_t(const hz_coeffs* cc, const void* b_in, void* x_in, int nrhs, const hz_solve_opts& o,
                  double* relres_out, int* iters_out, hz_solve_stats* stats, cudaStream_t s) {
  typedef typename Cx<R>::T C;
  hz_coeffs* c = const_cast<hz_coeffs*>(cc);
  const long long launches0 = g_launches.load();
  if (!c->work || c->work->nrhs != nrhs) c->work.reset(new SolverWork);
  SolverWork& w = *c->work;
  w.nrhs = nrhs;
  const size_t fb = (size_t)c->fstride() * nrhs * sizeof(C);
  HZ_CUDA(w.rhat.ensure(fb));
  HZ_CUDA(w.p.ensure(fb));
  HZ_CUDA(w.v.ensure(fb));
  HZ_CUDA(w.t.ensure(fb));
  HZ_CUDA(w.r.ensure(fb));
  const bool ell2 = o.ell == 2;
  if (ell2) {
    HZ_CUDA(w.r1.ensure(fb));
    HZ_CUDA(w.r2.ensure(fb));
    HZ_CUDA(w.dotG.ensure(sizeof(double) * nrhs));
  }
  if (sizeof(R) == 4) HZ_CUDA(w.xlo.ensure(fb));
  const bool pre = o.precond == 1 && sizeof(R) == 4;
  if (pre) {
    HZ_CUDA(w.ph.ensure(fb));
    HZ_CUDA(w.sh.ensure(fb));
  }
  // the workspace starts at zero: pad columns stay 0 in every Krylov vector (the applies write
  // zeros there, the fp64 residual does not touch them), so the flat dot products see only points
  for (DBuf* d : {&w.rhat, &w.p, &w.v, &w.t, &w.r, &w.r1, &w.r2, &w.xlo, &w.ph, &w.sh})
    if (d->p && d->n >= fb) HZ_CUDA(cudaMemsetAsync(d->p, 0, fb, s));
  HZ_CUDA(w.dotA.ensure(sizeof(double) * 2 * nrhs));
  HZ_CUDA(w.dotB.ensure(sizeof(double) * 7 * nrhs));
  HZ_CUDA(w.dotR.ensure(sizeof(double) * 3 * nrhs));
  HZ_CUDA(w.dotN.ensure(sizeof(double) * nrhs));
  HZ_CUDA(w.state.ensure(sizeof(SolverState) * nrhs));
  HZ_CUDA(w.active.ensure(sizeof(int) * nrhs));
  const long long n = c->plane() * c->grid.nz_local;   // storage elements of the owned planes (pads included)
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->ctx->device);
  const int vblocks = (int)std::max(1LL, std::min((n + 1023) / 1024, (long long)(8 * sms + nrhs - 1) / nrhs));
  HZ_CUDA(w.partials.ensure(sizeof(double) * (size_t)vblocks * nrhs * 3));   // ≤ 3 dots per vector kernel
  HZ_CUDA(w.tickets.ensure(sizeof(unsigned) * nrhs));
  HZ_CUDA(cudaMemsetAsync(w.tickets.p, 0, sizeof(unsigned) * nrhs, s));
  HZ_CUDA(cudaMemsetAsync(w.state.p, 0, sizeof(SolverState) * nrhs, s));
  // host / device placement of b and x
  const bool db = is_device_ptr(b_in), dx = is_device_ptr(x_in);
  const C* b = reinterpret_cast<const C*>(b_in);
  C* x = reinterpret_cast<C*>(x_in);
  if (!db) {
    HZ_CUDA(w.hb.ensure(fb));
    HZ_CUDA(cudaMemcpyAsync(w.hb.p, b_in, fb, cudaMemcpyHostToDevice, s));
    b = w.hb.as<C>();
  }
  if (!dx) {
    HZ_CUDA(w.hx.ensure(fb));
    HZ_CUDA(cudaMemcpyAsync(w.hx.p, x_in, fb, cudaMemcpyHostToDevice, s));
    x = w.hx.as<C>();
  }
  std::vector<int> active(nrhs, 1), iters(nrhs, 0);
  HZ_CUDA(cudaMemcpyAsync(w.active.p, active.data(), sizeof(int) * nrhs, cudaMemcpyHostToDevice, s));
  auto n_active = [&]() {
    int k = 0;
    for (int r = 0; r < nrhs; r++) k += active[r] != 0;
    return k;
  };

  EventTimer timer;
  timer.on = o.timing != 0;
  long long apply_launches = 0;
  double apply_bytes = 0.0, apply_points = 0.0;
  // algorithmic bytes of one apply launch: v (shared by the RHS) + per active RHS the fields
  // the epilogue touches (u in, out, plus r̂0 / b reads)
  auto account = [&](int nfields_per_rhs) {
    apply_bytes += (double)n * ((double)sizeof(R) + (double)n_active() * nfields_per_rhs * (double)sizeof(C));
    apply_points += (double)n * (double)n_active();
    apply_launches++;
  };
  ApplyParams<R> base = make_params<R>(c);
  base.active = w.active.as<int>();
  VecParams<R> q;
  memset(&q, 0, sizeof(q));
  q.n = n;
  q.plane = c->plane();
  q.fstride = c->fstride();
  q.nblocks = vblocks;
  q.x = x;
  q.r = w.r.as<C>();
  q.rhat = w.rhat.as<C>();
  q.p = w.p.as<C>();
  q.v = w.v.as<C>();
  q.t = w.t.as<C>();
  q.xlo = sizeof(R) == 4 ? w.xlo.as<C>() : nullptr;
  q.r1 = ell2 ? w.r1.as<C>() : nullptr;
  q.r2 = ell2 ? w.r2.as<C>() : nullptr;
  q.dotG = ell2 ? w.dotG.as<double>() : nullptr;
  q.dotA = w.dotA.as<double>();
  q.dotB = w.dotB.as<double>();
  q.dotR = w.dotR.as<double>();
  q.partials = w.partials.as<double>();
  q.tickets = w.tickets.as<unsigned>();
  q.state = w.state.as<SolverState>();
  q.active = w.active.as<int>();
  if constexpr (sizeof(R) == 4) {
    if (pre) {
      if (!w.mg) {
        MgSpec sp;
        sp.nx = c->grid.nx;
        sp.ny = c->grid.ny;
        sp.nz = c->grid.nz_local;
        sp.ldx = c->ldx;
        sp.plane = c->plane();
        sp.fstride = c->fstride();
        sp.w = c->w.as<float>();
        sp.h = c->h;
        sp.omega = c->omega;
        sp.beta = HZ_MG_BETA;
        sp.vmin = c->vmin;
        sp.vmax = c->vmax;
        sp.v_pml = c->v_pml;
        sp.r_coeff = c->pml.r_coeff;
        sp.npml = c->pml.npml;
        sp.nrhs = nrhs;
        sp.max_levels = 12;
        MgHierarchy* m = nullptr;
        HZ_CUDA(mg_create(sp, &m));
        w.mg.reset(m);
      }
      q.ph = w.ph.as<C>();
      q.sh = w.sh.as<C>();
    }
  }

  // r = b − A x (RESID epilogue; writes r, ‖r‖², (r̂0, r)).  For complex64 the residual is
  // computed in fp64 arithmetic on the c64 storage (reading A21): the fp32 apply's rounding
  // (~eps32·‖|A||x|‖/‖b‖ ≈ 1e-6 on config 1) would otherwise set the attainable true residual.
  bool use_lo = sizeof(R) == 4;   // false for the final residual of the rounded output x
  auto resid = [&](bool with_rhat) -> hz_status {
    HZ_TRY(halo_exchange(c, x, nrhs, sizeof(C), s));
    if (use_lo) HZ_TRY(halo_exchange(c, w.xlo.p, nrhs, sizeof(C), s));   // the compensation word's halo too
    timer.mark(s);
    if constexpr (sizeof(R) == 4) {
      ApplyParams<double, float> p = make_params<double, float>(c);
      p.active = w.active.as<int>();
      p.u = x;
      p.ulo = use_lo ? w.xlo.as<C>() : nullptr;
      p.au = w.r.as<C>();
      p.bvec = b;
      p.rhat = with_rhat ? w.rhat.as<C>() : nullptr;
      p.dots = w.dotR.as<double>();
      HZ_TRY(apply_launch<double, float>(c, p, nrhs, EPI_RESID, s));
    } else {
      ApplyParams<R> p = base;
      p.u = x;
      p.au = w.r.as<C>();
      p.bvec = b;
      p.rhat = with_rhat ? w.rhat.as<C>() : nullptr;
      p.dots = w.dotR.as<double>();
      HZ_TRY(apply_launch<R, R>(c, p, nrhs, EPI_RESID, s));
    }
    timer.mark(s);
    account((with_rhat ? 4 : 3) + (use_lo ? 1 : 0));
    HZ_TRY(allreduce_sum(c, w.dotR.as<double>(), 3 * (size_t)nrhs, s));
    return HZ_OK;
  };
  auto vec = [&](int which) -> hz_status {
    HZ_CUDA(launch_bicg<R>(which, q, nrhs, s));
    count_launch();
    return HZ_OK;
  };

  // ‖b‖²
  HZ_CUDA(launch_norm2<R>(b, c->fstride(), c->plane(), c->npoints(), c->grid.nx, c->ldx, nrhs, vblocks,
                          w.partials.as<double>(), w.dotN.as<double>(), w.tickets.as<unsigned>(), s));
  count_launch();
  HZ_TRY(allreduce_sum(c, w.dotN.as<double>(), nrhs, s));
  std::vector<double> bn2(nrhs);
  HZ_CUDA(cudaMemcpyAsync(bn2.data(), w.dotN.p, sizeof(double) * nrhs, cudaMemcpyDeviceToHost, s));
  HZ_CUDA(cudaStreamSynchronize(s));
  // RHS with b = 0: x = 0, converged
  for (int r = 0; r < nrhs; r++)
    if (!(bn2[r] > 0)) {
      active[r] = 0;
      HZ_CUDA(cudaMemsetAsync(x + (size_t)r * c->fstride(), 0, sizeof(C) * c->fstride(), s));
    }
  HZ_CUDA(cudaMemcpyAsync(w.active.p, active.data(), sizeof(int) * nrhs, cudaMemcpyHostToDevice, s));
  // complex64: iterate the double-word x + x_lo to rtol/2 so that the returned (rounded) x meets rtol
  // despite its own rounding floor (~eps32·‖|A||x|‖/‖b‖, 2–5e-7 on configs 1–3; reading A21)
  const double rtol_it = sizeof(R) == 4 ? 0.5 * o.rtol : o.rtol;
  const double rtol2 = rtol_it * rtol_it;
  auto init = [&]() -> hz_status {
    if (!ell2) return vec(BICG_INIT);
    HZ_CUDA(launch_bicgl<R>(BCL_INIT, q, nrhs, s));
    count_launch();
    return HZ_OK;
  };
  HZ_TRY(resid(false));
  HZ_TRY(init());

  int restarts = 0, replacements = 0;
  // breakdown restarts per RHS: a RHS that breaks down more than restart_cap times is retired on its
  // own (HZ_BREAKDOWN); the cap lets the stall window act first on a RHS at its rounding floor
  std::vector<int> rs_count(nrhs, 0);
  bool broke_any = false;
  int it = 0;
  std::vector<double> hdot(3 * nrhs);
  std::vector<SolverState> hst(nrhs);
  // stagnation guard: best true residual per RHS and the iteration it was reached
  std::vector<double> best(nrhs, HUGE_VAL);
  std::vector<int> best_it(nrhs, 0);
  bool stagnated_any = false;
  const int stall_iters = o.stall_window > 0   ? o.stall_window
                          : o.stall_window < 0 ? INT_MAX
                                               : std::max(20 * std::max(1, o.replace_every), 1000);
  const int restart_cap = std::max(50, stall_iters == INT_MAX ? INT_MAX / 2 : stall_iters / std::max(1, o.check_every) + 1);
  // initial convergence check (x0 may already solve the system)
  HZ_CUDA(cudaMemcpyAsync(hdot.data(), w.dotR.p, sizeof(double) * 3 * nrhs, cudaMemcpyDeviceToHost, s));
  HZ_CUDA(cudaStreamSynchronize(s));
  for (int r = 0; r < nrhs; r++)
    if (active[r] && hdot[3 * r] <= rtol2 * bn2[r]) active[r] = 0;
  HZ_CUDA(cudaMemcpyAsync(w.active.p, active.data(), sizeof(int) * nrhs, cudaMemcpyHostToDevice, s));

  // deactivate RHS whose TRUE residual (in hdot after a resid) meets rtol or has stagnated
  auto retire = [&](bool true_resid) -> hz_status {
    bool changed = false;
    for (int r = 0; r < nrhs; r++) {
      if (!active[r]) continue;
      if (hdot[3 * r] <= rtol2 * bn2[r]) {
        active[r] = 0;
        changed = true;
      } else if (true_resid) {
        if (hdot[3 * r] < 0.81 * best[r]) {   // ≥ 10% reduction of the norm
          best[r] = hdot[3 * r];
          best_it[r] = it;
        } else if (it - best_it[r] >= stall_iters) {
          active[r] = 0;
          changed = true;
          stagnated_any = true;
        }
      }
    }
    if (changed) HZ_CUDA(cudaMemcpyAsync(w.active.p, active.data(), sizeof(int) * nrhs, cudaMemcpyHostToDevice, s));
    return HZ_OK;
  };

  // one operator apply with a dot epilogue (+ the ranks' sum of its dots)
  auto apply_dots = [&](DBuf& in, DBuf& out, int epi, const C* rh, DBuf& dots, int ndots, const C* sdot = nullptr) -> hz_status {
    ApplyParams<R> p = base;
    p.u = in.as<C>();
    p.au = out.as<C>();
    p.rhat = rh;
    p.bvec = sdot;   // DOT4 operand s when it is not the input (right preconditioning)
    p.dots = dots.as<double>();
    timer.mark(s);
    HZ_TRY(apply_launch<R, R>(c, p, nrhs, epi, s, true));   // halo exchange overlapped with the interior
    timer.mark(s);
    account(3);
    HZ_TRY(allreduce_sum(c, dots.as<double>(), (size_t)ndots * nrhs, s));
    return HZ_OK;
  };
  auto vecl = [&](int which) -> hz_status {
    HZ_CUDA(launch_bicgl<R>(which, q, nrhs, s));
    count_launch();
    return HZ_OK;
  };
  // after a residual replacement: BiCGSTAB re-reads ρ = (r̂0, r) from dotR; BiCGStab(2) always does
  auto rho_reset = [&]() -> hz_status { return ell2 ? HZ_OK : vec(BICG_RHO_RESET); };
  const C* rh = w.rhat.as<C>();

  while (n_active() > 0 && it < o.max_iter) {
    int inc = 1;
    if (!ell2 && pre) {   // right preconditioning (A27): v = A M⁻¹p, t = A M⁻¹s, x += α M⁻¹p + ω M⁻¹s
      if constexpr (sizeof(R) == 4) {
        long long nl = 0;
        HZ_CUDA(mg_vcycle(w.mg.get(), w.p.as<float2>(), w.ph.as<float2>(), nrhs, w.active.as<int>(), s, &nl));
        count_launch(nl);
        HZ_TRY(apply_dots(w.ph, w.v, EPI_DOT1, rh, w.dotA, 2));
        HZ_TRY(vec(BICG_S));
        nl = 0;
        HZ_CUDA(mg_vcycle(w.mg.get(), w.r.as<float2>(), w.sh.as<float2>(), nrhs, w.active.as<int>(), s, &nl));
        count_launch(nl);
        HZ_TRY(apply_dots(w.sh, w.t, EPI_DOT4, rh, w.dotB, 7, w.r.as<C>()));   // (t,s) with s, not M⁻¹s
        HZ_TRY(vec(BICG_UPDATE));
      }
      HZ_TRY(allreduce_sum(c, w.dotR.as<double>(), 3 * (size_t)nrhs, s));
    } else if (!ell2) {
      HZ_TRY(apply_dots(w.p, w.v, EPI_DOT1, rh, w.dotA, 2));   // v = A p, (r̂0, v)
      HZ_TRY(vec(BICG_S));                                      // s = r − α v (in r)
      HZ_TRY(apply_dots(w.r, w.t, EPI_DOT4, rh, w.dotB, 7));   // t = A s, (t,s), (t,t), (r̂0,s), (r̂0,t)
      HZ_TRY(vec(BICG_UPDATE));                                 // x, r, p; ‖r‖²
      HZ_TRY(allreduce_sum(c, w.dotR.as<double>(), 3 * (size_t)nrhs, s));
    } else {   // one BiCGStab(2) outer step (kernels.cu K3'): four applies = two BiCGSTAB iterations
      inc = 2;
      HZ_TRY(vecl(BCL_A));
      HZ_TRY(apply_dots(w.p, w.v, EPI_DOT1, rh, w.dotA, 2));   // u1 = A u0
      HZ_TRY(vecl(BCL_B));
      HZ_TRY(apply_dots(w.r, w.r1, EPI_DOT1, rh, w.dotA, 2));  // r1 = A r0
      HZ_TRY(vecl(BCL_C));
      HZ_TRY(apply_dots(w.v, w.t, EPI_DOT1, rh, w.dotA, 2));   // u2 = A u1
      HZ_TRY(vecl(BCL_D));
      HZ_TRY(allreduce_sum(c, w.dotG.as<double>(), (size_t)nrhs, s));
      HZ_TRY(apply_dots(w.r1, w.r2, EPI_DOT4, w.r.as<C>(), w.dotB, 7));   // r2 = A r1 (r̂ := r0)
      HZ_TRY(vecl(BCL_E));
      HZ_TRY(allreduce_sum(c, w.dotR.as<double>(), 3 * (size_t)nrhs, s));
    }
    it += inc;
    for (int r = 0; r < nrhs; r++)
      if (active[r]) iters[r] += inc;
    auto crossed = [&](int period) { return period > 0 && it / period > (it - inc) / period; };
    const bool replaced = crossed(o.replace_every);
    if (replaced) {
      HZ_TRY(resid(true));
      HZ_TRY(rho_reset());
      replacements++;
    }
    if (replaced || crossed(std::max(1, o.check_every)) || it >= o.max_iter) {
      HZ_CUDA(cudaMemcpyAsync(hdot.data(), w.dotR.p, sizeof(double) * 3 * nrhs, cudaMemcpyDeviceToHost, s));
      HZ_CUDA(cudaMemcpyAsync(hst.data(), w.state.p, sizeof(SolverState) * nrhs, cudaMemcpyDeviceToHost, s));
      HZ_CUDA(cudaStreamSynchronize(s));
      bool cand = false, brk = false;
      for (int r = 0; r < nrhs; r++) {
        if (!active[r]) continue;
        if (hst[r].flags & 1) {
          brk = true;
          if (++rs_count[r] > restart_cap) {   // this RHS alone is retired
            active[r] = 0;
            broke_any = true;
          }
        } else if (hdot[3 * r] <= rtol2 * bn2[r]) {
          cand = true;
        }
      }
      if (brk) {  // restart broken RHS with r̂0 = r = b − A x (all active RHS restart together)
        HZ_CUDA(cudaMemcpyAsync(w.active.p, active.data(), sizeof(int) * nrhs, cudaMemcpyHostToDevice, s));
        if (n_active() == 0) break;
        HZ_TRY(resid(false));
        // the recomputed true residuals also feed the convergence / stagnation test, so a RHS at its
        // rounding floor (where breakdowns recur) is retired by the stall window, not the restart cap
        HZ_CUDA(cudaMemcpyAsync(hdot.data(), w.dotR.p, sizeof(double) * 3 * nrhs, cudaMemcpyDeviceToHost, s));
        HZ_CUDA(cudaStreamSynchronize(s));
        HZ_TRY(retire(true));
        HZ_TRY(init());
        restarts++;
        continue;
      }
      if (replaced) {
        HZ_TRY(retire(true));           // hdot holds the recomputed true residuals
      } else if (cand) {                // verify on the recomputed TRUE residual (A21)
        HZ_TRY(resid(true));
        HZ_TRY(rho_reset());
        replacements++;
        HZ_CUDA(cudaMemcpyAsync(hdot.data(), w.dotR.p, sizeof(double) * 3 * nrhs, cudaMemcpyDeviceToHost, s));
        HZ_CUDA(cudaStreamSynchronize(s));
        HZ_TRY(retire(true));
      }
    }
  }
  // final true residuals for every RHS, of the output x itself (the rounded double-word iterate)
  use_lo = false;
  std::vector<int> all(nrhs, 1);
  active = all;
  HZ_CUDA(cudaMemcpyAsync(w.active.p, all.data(), sizeof(int) * nrhs, cudaMemcpyHostToDevice, s));
  HZ_TRY(resid(false));
  HZ_CUDA(cudaMemcpyAsync(hdot.data(), w.dotR.p, sizeof(double) * 3 * nrhs, cudaMemcpyDeviceToHost, s));
  HZ_CUDA(cudaStreamSynchronize(s));
  bool conv = true;
  for (int r = 0; r < nrhs; r++) {
    const double rel = bn2[r] > 0 ? std::sqrt(hdot[3 * r] / bn2[r]) : 0.0;   // of the returned x
    if (relres_out) relres_out[r] = rel;
    if (iters_out) iters_out[r] = iters[r];
    if (!(rel <= o.rtol)) conv = false;
  }
  if (!dx) {
    HZ_CUDA(cudaMemcpyAsync(x_in, x, fb, cudaMemcpyDeviceToHost, s));
    HZ_CUDA(cudaStreamSynchronize(s));
  }
  if (stats) {
    stats->apply_ms_total = timer.on ? timer.total_ms() : 0.0;
    stats->apply_launches = apply_launches;
    stats->kernel_launches = g_launches.load() - launches0;
    stats->apply_bytes_total = apply_bytes;
    stats->apply_points_total = apply_points;
    stats->replacements = replacements;
    stats->restarts = restarts;
    stats->iterations = it;
    stats->stagnated = stagnated_any ? 1 : 0;
  }
  if (conv) return HZ_OK;
  return broke_any ? HZ_BREAKDOWN : HZ_NOT_CONVERGED;
}

}  // namespace

extern "C" hz_solve_opts hz_solve_opts_default(void) {
  hz_solve_opts o;
  memset(&o, 0, sizeof(o));
  o.rtol = 1e-6;
  o.max_iter = 20000;
  o.replace_every = 50;
  o.check_every = 10;
  o.ell = 1;
  return o;
}

extern "C" hz_status hz_solve(const hz_coeffs* c, const void* b, void* x, int nrhs, const hz_solve_opts* opts,
                              double* relres_out, int* iters_out, hz_solve_stats* stats, void* stream) {
  if (!c || !b || !x || nrhs < 1) { set_error("hz_solve: bad arguments"); return HZ_ERR_INVALID_ARG; }
  HZ_TRY(set_device(c->ctx));
  hz_solve_opts o = hz_solve_opts_default();
  if (opts) o = *opts;
  // zero selects each field's default (a zero-initialised struct is the default configuration)
  if (o.rtol == 0) o.rtol = 1e-6;
  if (o.max_iter == 0) o.max_iter = 20000;
  if (o.replace_every == 0) o.replace_every = 50;
  if (o.check_every == 0) o.check_every = 10;
  if (!(o.rtol > 0) || o.max_iter < 1) { set_error("hz_solve: need rtol > 0, max_iter >= 1"); return HZ_ERR_INVALID_ARG; }
  if (o.replace_every < 0) o.replace_every = 0;   // < 0: no residual replacement
  if (o.check_every < 1) { set_error("hz_solve: check_every must be >= 0"); return HZ_ERR_INVALID_ARG; }
  if (o.ell == 0) o.ell = 1;
  if (o.ell != 1 && o.ell != 2) { set_error("hz_solve: ell must be 1 (BiCGSTAB) or 2 (BiCGStab(2))"); return HZ_ERR_INVALID_ARG; }
  if (o.precond != 0 && o.precond != 1) { set_error("hz_solve: precond must be 0 or 1"); return HZ_ERR_INVALID_ARG; }
  if (o.precond == 1 && (c->dtype != HZ_C64 || o.ell != 1 || c->ctx->nranks != 1 || c->medium || c->grid.nz_local != c->grid.nz_global)) {
    set_error("hz_solve: the multigrid preconditioner needs complex64, ell = 1, one rank and the acoustic (rho = 1) operator");
    return HZ_ERR_INVALID_ARG;
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  return c->dtype == HZ_C64 ? solve_t<float>(c, b, x, nrhs, o, relres_out, iters_out, stats, s)
                            : solve_t<double>(c, b, x, nrhs, o, relres_out, iters_out, stats, s);
}
