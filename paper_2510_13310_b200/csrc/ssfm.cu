// ssfm.cu -- C-ABI (include/ssfm.h) and host drivers of the B200-native
// sparse LM core. One translation unit: the kernels live in the .cuh files.
//
// Host side of lm_solve (lm.py:727-800) is a plain C++ loop that launches the
// device pipeline and reads back ONE small status block per LM iteration
// (status bits, CG iteration count, candidate cost, gradient max); everything
// else (linearize, J^T r, elimination, PCG, back-substitution, update, cost)
// stays on the device.
#include <cuda_runtime.h>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <algorithm>
#include <initializer_list>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ssfm.h"
#include "ba_pcg.cuh"
#include "ba_pcg_graph.cuh"
#include "gp_pcg_graph.cuh"
#include "gp_kernels.cuh"
#include "pattern.cuh"
#include "block_algebra.cuh"
#include "dense.cuh"
#include "lm_graph.cuh"
#include "prune.cuh"
#include "schur_explicit.cuh"
#include "metrics.cuh"

static thread_local std::string g_last_error;

static int set_err(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

// error hand-off for the host-only translation units (bal_host.cpp)
extern "C" int ssfm_internal_set_error(int code, const char* msg) { return set_err(code, msg ? msg : ""); }

#define CU(call)                                                                   \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess)                                                         \
      return set_err(SSFM_CUDA_ERROR, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

struct Misc {
  int status;
  int pad;
  double scal[8];
  CGCtl ctl;
};

struct Profile {
  bool on = false;
  double phase_ms[5] = {0, 0, 0, 0, 0};
  double pcg_ms = 0, lin_ms = 0, all_ms = 0;
  long long pcg_launches = 0, lin_launches = 0, all_launches = 0;
  long long cg_iters = 0;
  long long kernel_launches = 0;   // every kernel launched by the library
};

// Grow-only device arena (the reference's Workspace, lm.py:86-101, as HBM):
// handles created in it (ssfm_create_ba_in / ssfm_create_gp_in) bump-allocate
// from its chunks and give nothing back one by one; when the last live handle
// is destroyed the arena is reset, so the next stage's handle (GP -> BA)
// reuses the same HBM without cudaMalloc. A stage that needs more than the
// arena holds adds a chunk; after a reset the chunks are coalesced into one of
// the high-water size (grow-only).
struct ssfm_arena {
  int device = 0;
  std::mutex mu;
  std::vector<std::pair<char*, size_t>> chunks;   // (base, bytes)
  size_t cur = 0;          // chunk being filled
  size_t off = 0;          // bytes used in chunks[cur]
  size_t used = 0;         // bytes handed out since the last reset
  size_t high_water = 0;
  int live = 0;            // handles holding allocations
  long long chunk_mallocs = 0;
};

static size_t arena_capacity(const ssfm_arena* a) {
  size_t s = 0;
  for (const auto& c : a->chunks) s += c.second;
  return s;
}

static int arena_alloc(ssfm_arena* a, size_t b, void** out) {
  std::lock_guard<std::mutex> lk(a->mu);
  if (a->live == 0 && a->used == 0 && a->chunks.size() > 1) {
    // coalesce the chunks of an idle arena into one of the high-water size
    const size_t total = std::max(arena_capacity(a), a->high_water);
    for (auto& c : a->chunks) cudaFree(c.first);
    a->chunks.clear();
    char* p = nullptr;
    if (cudaMalloc((void**)&p, total) != cudaSuccess) {
      cudaGetLastError();
      return set_err(SSFM_CUDA_ERROR, "arena: cudaMalloc failed while coalescing");
    }
    a->chunks.emplace_back(p, total);
    a->chunk_mallocs++;
    a->cur = 0;
    a->off = 0;
  }
  while (a->cur < a->chunks.size() && a->off + b > a->chunks[a->cur].second) {
    ++a->cur;
    a->off = 0;
  }
  if (a->cur >= a->chunks.size()) {
    const size_t grow = std::max(b, std::max(arena_capacity(a), (size_t)256 << 20));
    char* p = nullptr;
    cudaError_t e = cudaMalloc((void**)&p, grow);
    if (e == cudaErrorMemoryAllocation && grow > b) {
      cudaGetLastError();
      e = cudaMalloc((void**)&p, b);
      if (e == cudaSuccess) a->chunks.emplace_back(p, b);
    } else if (e == cudaSuccess) {
      a->chunks.emplace_back(p, grow);
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      return set_err(SSFM_CUDA_ERROR, std::string("arena: cudaMalloc: ") + cudaGetErrorString(e));
    }
    a->chunk_mallocs++;
    a->cur = a->chunks.size() - 1;
    a->off = 0;
  }
  *out = a->chunks[a->cur].first + a->off;
  a->off += b;
  a->used += b;
  a->high_water = std::max(a->high_water, a->used);
  return SSFM_OK;
}

static void arena_release(ssfm_arena* a) {
  std::lock_guard<std::mutex> lk(a->mu);
  if (--a->live == 0) {
    a->cur = 0;
    a->off = 0;
    a->used = 0;
  }
}

struct ssfm_handle {
  int kind = 0;   // 0 BA, 1 GP
  int device = 0;
  int num_sms = 148;
  int pcg_sms = 148;            // SMs the persistent PCG grid may occupy (SSFM_PCG_SMS)
  std::vector<void*> allocs;
  size_t bytes = 0;
  long long total_params = 0, total_res = 0;
  BADev ba{};
  GPDev gp{};
  Topo topo{};
  // solver state
  double *theta = nullptr, *cand = nullptr, *delta = nullptr;
  double *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
  double* part = nullptr;       // PCG per-CTA partials
  double* red = nullptr;        // reduction scratch (cost / gnorm)
  long long red_n = 0;
  Misc* misc = nullptr;         // device
  Misc* hmisc = nullptr;        // pinned host
  int pcg_grid = 0;
  int pcg_threads = PCG_THREADS;
  size_t pcg_smem = 0;
  void* pcg_fn = nullptr;
  FusedTopo fz{};
  // point sharding (comm.cuh)
  CommDev cm{};
  void* region = nullptr;
  std::vector<void*> ipc_opened;
  double* camsum = nullptr;     // [CAM_V * C] per-camera sums exchanged between ranks
  double* ar_tmp = nullptr;     // [16] scalar scratch
  int comm_nranks = 1;
  // graph PCG (ba_pcg_graph.cuh): built on first use, reused for every solve
  int graph_state = 0;          // 0 not built, 1 ready, -1 unavailable (persistent kernel)
  bool graph_sharded = false;   // the built graph carries the exchange kernels
  bool graph_pending = false;   // a graph solve whose body kernels are not yet counted
  int graph_body_kernels = 0;   // kernels per WHILE-body iteration
  cudaGraph_t pcg_graph = nullptr;
  cudaGraphExec_t pcg_exec = nullptr;
  CGGraphDev gdev{};
  int lin_blocks = 0;
  int cost_blocks = 0;
  int cam_blocks = 0;
  bool linearized = false;
  Profile prof;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
  std::vector<size_t> alloc_bytes;   // sizes of allocs (block cache)
  ssfm_arena* arena = nullptr;       // allocations come from this arena (not from allocs)
  // the LM loop as one CUDA graph (lm_graph.cuh): built on the first lm_solve
  int lm_state = 0;             // 0 not built, 1 ready, -1 unavailable (host loop)
  cudaGraph_t lm_graph = nullptr;
  cudaGraphExec_t lm_exec = nullptr;
  LMState* lms = nullptr;       // device
  LMState* hlms = nullptr;      // pinned host
  LMRecDev* lrecs = nullptr;    // device [lrec_cap]
  LMRecDev* hlrecs = nullptr;   // pinned host
  int lrec_cap = 0;
  double* lm_theta = nullptr;   // the theta buffer the graph was captured with
  double lm_cg_tol = -1.0;      // CG parameters baked into the captured PCG launches
  int lm_cg_max = -1;
  long long lm_k_iter = 0, lm_k_lin = 0, lm_k_solve = 0;   // kernels per section (launch accounting)
  bool capturing = false;
};

// Device blocks of destroyed handles are kept for reuse by exact size (per
// device, up to SSFM_BLOCK_CACHE_GB, default 48): re-creating a handle of the
// same shape -- repeated solves, the GP -> BA pipeline, the e2e bench -- skips
// cudaMalloc / cudaFree, whose page mapping and implicit device syncs cost
// 40-190 ms at C5. Guarded by a mutex (handles may be created from several
// host threads).
struct BlockCache {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> free_blocks;   // (device, bytes) -> block
  size_t bytes = 0;
};
static BlockCache& block_cache() {
  static BlockCache c;
  return c;
}
// cap: SSFM_BLOCK_CACHE_GB, else a quarter of the device's HBM
static size_t block_cache_cap() {
  const char* e = getenv("SSFM_BLOCK_CACHE_GB");
  if (e) return (size_t)(atof(e) * (double)(1ull << 30));
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) return 0;
  return tot / 4;
}

// free the cached blocks of `device` (-1: every device); returns bytes freed
static size_t block_cache_trim(int device) {
  BlockCache& bc = block_cache();
  std::lock_guard<std::mutex> lk(bc.mu);
  size_t freed = 0;
  for (auto it = bc.free_blocks.begin(); it != bc.free_blocks.end();) {
    if (device < 0 || it->first.first == device) {
      cudaFree(it->second);
      freed += it->first.second;
      bc.bytes -= it->first.second;
      it = bc.free_blocks.erase(it);
    } else {
      ++it;
    }
  }
  return freed;
}

template <typename T>
static int dalloc(ssfm_handle* h, T** ptr, size_t count) {
  size_t b = sizeof(T) * (count > 0 ? count : 1);
  b = (b + 255) & ~size_t(255);
  void* p = nullptr;
  if (h->arena) {
    const int rc = arena_alloc(h->arena, b, &p);
    if (rc) return rc;
    h->bytes += b;
    *ptr = static_cast<T*>(p);
    return SSFM_OK;
  }
  {
    BlockCache& bc = block_cache();
    std::lock_guard<std::mutex> lk(bc.mu);
    auto it = bc.free_blocks.find({h->device, b});
    if (it != bc.free_blocks.end()) {
      p = it->second;
      bc.free_blocks.erase(it);
      bc.bytes -= b;
    }
  }
  if (!p) {
    cudaError_t e = cudaMalloc(&p, b);
    if (e == cudaErrorMemoryAllocation && block_cache_trim(h->device) > 0) {
      cudaGetLastError();   // clear the failed allocation, retry with the cache released
      e = cudaMalloc(&p, b);
    }
    if (e != cudaSuccess)
      return set_err(SSFM_CUDA_ERROR, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  }
  h->allocs.push_back(p);
  h->alloc_bytes.push_back(b);
  h->bytes += b;
  *ptr = static_cast<T*>(p);
  return SSFM_OK;
}

#define DALLOC(ptr, n)                        \
  do {                                        \
    int _rc = dalloc(h, &(ptr), (size_t)(n)); \
    if (_rc) return _rc;                      \
  } while (0)

static inline int nblk(long long n, int t) { return (int)((n + t - 1) / t); }

// zero / copy on the stream as kernels (see k_fill_u32 in common.cuh)
static cudaError_t zero_async(void* p, size_t bytes, cudaStream_t st) {
  const long long n = (long long)(bytes / 4);
  k_fill_u32<<<std::max(1, std::min(nblk(n, 256), 1184)), 256, 0, st>>>(static_cast<unsigned*>(p), n, 0u);
  return cudaGetLastError();
}
static cudaError_t copy_async(double* dst, const double* src, long long n, cudaStream_t st) {
  k_copy_f64<<<std::max(1, std::min(nblk(n, 256), 1184)), 256, 0, st>>>(dst, src, n);
  return cudaGetLastError();
}

static void free_handle(ssfm_handle* h) {
  if (!h) return;
  for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
  if (h->pcg_exec) cudaGraphExecDestroy(h->pcg_exec);
  if (h->pcg_graph) cudaGraphDestroy(h->pcg_graph);
  if (!h->allocs.empty()) {
    // no kernel may still use the blocks (cudaFree synchronized implicitly)
    cudaDeviceSynchronize();
    BlockCache& bc = block_cache();
    const size_t cap = block_cache_cap();
    std::lock_guard<std::mutex> lk(bc.mu);
    for (size_t k = 0; k < h->allocs.size(); ++k) {
      const size_t b = h->alloc_bytes[k];
      if (bc.bytes + b <= cap) {
        bc.free_blocks.emplace(std::make_pair(h->device, b), h->allocs[k]);
        bc.bytes += b;
      } else {
        cudaFree(h->allocs[k]);
      }
    }
  }
  if (h->arena) {
    cudaDeviceSynchronize();   // no kernel may still use the arena's bytes
    arena_release(h->arena);
  }
  if (h->region) cudaFree(h->region);
  if (h->hmisc) cudaFreeHost(h->hmisc);
  if (h->hlms) cudaFreeHost(h->hlms);
  if (h->hlrecs) cudaFreeHost(h->hlrecs);
  if (h->lm_exec) cudaGraphExecDestroy(h->lm_exec);
  if (h->lm_graph) cudaGraphDestroy(h->lm_graph);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->ev2) cudaEventDestroy(h->ev2);
  if (h->ev3) cudaEventDestroy(h->ev3);
  delete h;
}

// ---------------------------------------------------------------------------
// topology build (shared by BA and GP)
// ---------------------------------------------------------------------------
static int build_topo(ssfm_handle* h, const int* cam, const int* pt, int C, int P, long long N,
                      cudaStream_t st, int* dstatus) {
  Topo& T = h->topo;
  T.C = C; T.P = P; T.N = N;
  const int TB = 256;
  CU(cudaMemsetAsync(dstatus, 0, sizeof(int), st));
  if (N > 0) k_check_index<<<nblk(N, TB), TB, 0, st>>>(cam, pt, N, C, P, dstatus);
  int hst = 0;
  CU(cudaMemcpyAsync(&hst, dstatus, sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (hst & ST_BAD_INDEX) return set_err(SSFM_INVALID_ARGUMENT, "observation references a camera or point index out of range");

  int *iota, *perm_pm, *perm_cm, *keys_out, *inv_cm, *cnt;
  DALLOC(iota, N); DALLOC(keys_out, N); DALLOC(inv_cm, N);
  DALLOC(T.pm_obs, N); DALLOC(T.cm_obs, N);
  // pm_pt / pm_cam + 4: 16-byte bulk copies of a batch's indices may round up past N
  DALLOC(T.pm_pt, N + 4); DALLOC(T.pm_cam, N + 4); DALLOC(T.pm_to_cm, N); DALLOC(T.cm_to_pm, N); DALLOC(T.cm_pt, N);
  DALLOC(T.pt_seg, (long long)P + 1); DALLOC(T.cam_seg, (long long)C + 1);
  perm_pm = T.pm_obs; perm_cm = T.cm_obs;
  if (N > 0) k_iota<<<nblk(N, TB), TB, 0, st>>>(iota, N);

  auto nbits = [](int n) { int b = 1; while ((1ll << b) < n) ++b; return b; };
  // stable radix sorts (point-major / camera-major)
  size_t tmp_bytes = 0, tb2 = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, pt, keys_out, iota, perm_pm, (int)N, 0, nbits(P), st);
  cub::DeviceRadixSort::SortPairs(nullptr, tb2, cam, keys_out, iota, perm_cm, (int)N, 0, nbits(C), st);
  tmp_bytes = std::max(tmp_bytes, tb2);
  size_t scan_bytes = 0;
  int maxPC = std::max(P, C) + 1;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, (int*)nullptr, (int*)nullptr, maxPC, st);
  tmp_bytes = std::max(tmp_bytes, scan_bytes);
  void* tmp;
  DALLOC(*(char**)&tmp, tmp_bytes);
  // stable sorts; segment offsets from the sorted keys (no atomics)
  if (N > 0) {
    CU(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, pt, keys_out, iota, perm_pm, (int)N, 0, nbits(P), st));
    k_seg_from_sorted<<<nblk(N, TB), TB, 0, st>>>(keys_out, N, P, T.pt_seg);
    CU(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, cam, keys_out, iota, perm_cm, (int)N, 0, nbits(C), st));
    k_seg_from_sorted<<<nblk(N, TB), TB, 0, st>>>(keys_out, N, C, T.cam_seg);
  }
  DALLOC(cnt, maxPC);
  if (N > 0) {
    k_perm_views<<<nblk(N, TB), TB, 0, st>>>(perm_pm, perm_cm, cam, pt, N, T.pm_pt, T.pm_cam, T.cm_pt, inv_cm);
    k_pm_to_cm<<<nblk(N, TB), TB, 0, st>>>(perm_pm, inv_cm, N, T.pm_to_cm);
    k_invert_perm<<<nblk(N, TB), TB, 0, st>>>(T.pm_to_cm, N, T.cm_to_pm);
  }
  // point batches
  int nch = nblk(P, SSFM_CHUNK);
  int *ch_cnt, *ch_off;
  DALLOC(ch_cnt, nch + 1); DALLOC(ch_off, nch + 1);
  CU(cudaMemsetAsync(ch_cnt, 0, sizeof(int) * (nch + 1), st));
  if (nch) k_batches<<<nblk(nch, 128), 128, 0, st>>>(T.pt_seg, P, 0, ch_cnt, ch_off, nullptr, nullptr);
  CU(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, ch_cnt, ch_off, nch + 1, st));
  int nb = 0;
  CU(cudaMemcpyAsync(&nb, ch_off + nch, sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  T.nb = nb;
  DALLOC(T.bat_pt, nb + 1); DALLOC(T.bat_obs, nb + 1);
  if (nch) k_batches<<<nblk(nch, 128), 128, 0, st>>>(T.pt_seg, P, 1, ch_cnt, ch_off, T.bat_pt, T.bat_obs);
  k_set_last<<<1, 1, 0, st>>>(T.bat_pt, nb, P);
  k_set_last<<<1, 1, 0, st>>>(T.bat_obs, nb, (int)N);
  // camera tiles
  DALLOC(T.cam_tile, C + 1);
  CU(cudaMemsetAsync(cnt, 0, sizeof(int) * maxPC, st));
  if (C) k_tile_count<<<nblk(C, TB), TB, 0, st>>>(T.cam_seg, C, cnt);
  CU(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, T.cam_tile, C + 1, st));
  int nt = 0;
  CU(cudaMemcpyAsync(&nt, T.cam_tile + C, sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  T.nt = nt;
  DALLOC(T.tile_obs, nt + 1); DALLOC(T.tile_cam, nt + 1);
  if (C) k_tile_write<<<nblk(C, TB), TB, 0, st>>>(T.cam_seg, T.cam_tile, C, T.tile_obs, T.tile_cam);
  k_set_last<<<1, 1, 0, st>>>(T.tile_obs, nt, (int)N);
  // tile groups (host: C + 1 tile offsets)
  {
    std::vector<int> ct(C + 1);
    CU(cudaMemcpyAsync(ct.data(), T.cam_tile, sizeof(int) * (C + 1), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    std::vector<int> g;
    for (int c = 0; c < C; ++c)
      for (int t = ct[c]; t < ct[c + 1]; t += SSFM_GRP) g.push_back(t);
    g.push_back(nt);
    T.ng = (int)g.size() - 1;
    DALLOC(T.grp_tile, g.size());
    CU(cudaMemcpyAsync(T.grp_tile, g.data(), sizeof(int) * g.size(), cudaMemcpyHostToDevice, st));
    CU(cudaStreamSynchronize(st));
  }
  CU(cudaGetLastError());
  return SSFM_OK;
}

// permute an interleaved [N,w] double array into point-major order
__global__ void k_gather_rows(const double* __restrict__ src, const int* __restrict__ perm, long long n,
                              int w, double* dst) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n) {
    const long long o = perm[i];
    for (int k = 0; k < w; ++k) dst[i * w + k] = src[o * w + k];
  }
}

static int common_alloc(ssfm_handle* h, int S_slots, int C) {
  DALLOC(h->theta, h->total_params);
  DALLOC(h->cand, h->total_params);
  DALLOC(h->delta, h->total_params);
  DALLOC(h->x, S_slots); DALLOC(h->r, S_slots); DALLOC(h->z, S_slots);
  DALLOC(h->p, S_slots); DALLOC(h->q, S_slots);
  DALLOC(h->misc, 1);
  CU(cudaMallocHost((void**)&h->hmisc, sizeof(Misc)));
  CU(cudaEventCreate(&h->ev0)); CU(cudaEventCreate(&h->ev1));
  CU(cudaEventCreate(&h->ev2)); CU(cudaEventCreate(&h->ev3));
  (void)C;
  return SSFM_OK;
}

// SSFM_PCG_SMS caps the SMs of the persistent PCG grid (several sharded
// handles on one device must be co-resident: their kernels wait on each other)
static int pcg_sms_of(const ssfm_handle* h) {
  if (const char* e = getenv("SSFM_PCG_SMS")) {
    const int v = atoi(e);
    if (v > 0 && v < h->num_sms) return v;
  }
  return h->num_sms;
}

// Choose the BA PCG operator and its launch geometry; build the fused schedule.
template <int SL>
static int try_fused_ba(ssfm_handle* h, int* ok) {
  *ok = 0;
  const int C = h->ba.bp.C;
  cudaFuncAttributes fa;
  CU(cudaFuncGetAttributes(&fa, ba_k_pcg<SL>));
  int optin = 0;
  CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
  const size_t dyn = sizeof(double) * ((size_t)SL * C + FZ_WARPS * 32 * SL) + sizeof(int) * (size_t)C;
  if (fa.sharedSizeBytes + dyn > (size_t)optin) return SSFM_OK;
  CU(cudaFuncSetAttribute(ba_k_pcg<SL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
  int occ = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ba_k_pcg<SL>, FZ_THREADS, dyn));
  if (occ < 1) return SSFM_OK;
  const int G = 8 / SL;
  int grid = occ * h->pcg_sms;
  grid -= grid % G;
  if (grid < G) return SSFM_OK;
  h->pcg_grid = grid;
  h->pcg_threads = FZ_THREADS;
  h->pcg_smem = dyn;
  h->pcg_fn = (void*)ba_k_pcg<SL>;
  h->fz.G = G;
  h->fz.SL = SL;
  h->fz.ngrp = grid / G;
  *ok = 1;
  return SSFM_OK;
}

// Ticket schedule of the fused operator (fused.cuh): stable sort of the
// observations by (CTA group, camera), runs walked in order. gpart gets
// `slots` doubles per camera per CTA group. *ok = 0 (fz cleared) when a camera
// has more than FZ_MAX_TICKET units in one group: use the two-pass operator.
static int build_fused_schedule(ssfm_handle* h, int slots, int* status, cudaStream_t st, int* ok) {
  const Topo& T = h->topo;
  FusedTopo& fz = h->fz;
  const int C = T.C;
  CU(cudaMemsetAsync(status, 0, sizeof(int), st));
  fz.nsteps = nblk(T.nb, FZ_WARPS);
  DALLOC(fz.tick, T.N);
  DALLOC(fz.gpart, (long long)fz.ngrp * slots * C);
  unsigned long long *key, *skey;
  int *unit, *idx, *sidx;
  std::vector<void*> tmp;
  auto talloc = [&](void** p, size_t b) { cudaError_t e = cudaMalloc(p, b); if (!e) tmp.push_back(*p); return e; };
  auto tfree = [&]() { cudaStreamSynchronize(st); for (void* q : tmp) cudaFree(q); };
  const long long N = T.N;
  if (talloc((void**)&key, 8 * N) || talloc((void**)&skey, 8 * N) || talloc((void**)&unit, 4 * N) ||
      talloc((void**)&idx, 4 * N) || talloc((void**)&sidx, 4 * N)) {
    tfree();
    return set_err(SSFM_CUDA_ERROR, "fused schedule: out of device memory");
  }
  k_fz_keys<<<nblk((long long)T.nb * 32, 256), 256, 0, st>>>(T, fz.ngrp, key, unit, idx);
  int kbits = 1;
  while ((1ull << kbits) < (unsigned long long)fz.ngrp * C) ++kbits;
  size_t sb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sb, key, skey, idx, sidx, (int)N, 0, kbits, st);
  void* stmp = nullptr;
  if (talloc(&stmp, sb)) { tfree(); return set_err(SSFM_CUDA_ERROR, "fused schedule: out of device memory"); }
  cub::DeviceRadixSort::SortPairs(stmp, sb, key, skey, idx, sidx, (int)N, 0, kbits, st);
  k_fz_tickets<<<nblk(N, 256), 256, 0, st>>>(skey, sidx, unit, N, fz.tick, status);
  int hst = 0;
  cudaMemcpyAsync(&hst, status, sizeof(int), cudaMemcpyDeviceToHost, st);
  tfree();
  *ok = 1;
  if (hst & ST_SCHEDULE) {
    h->fz = FusedTopo{};
    cudaMemsetAsync(status, 0, sizeof(int), st);
    *ok = 0;
  }
  CU(cudaGetLastError());
  return SSFM_OK;
}

static int setup_ba_pcg_op(ssfm_handle* h, cudaStream_t st);
// GP PCG operator. Default: the two-pass operator, as a CUDA graph from 250k
// observations (single-rank), else the persistent kernel. Measured (1xB200,
// ms per CG iteration): C4 GP 4M obs -- graph two-pass 0.137, fused persistent
// 0.158, two-pass persistent 0.175; C2 GP 300k obs -- 0.035 either two-pass,
// fused 0.042. SSFM_FUSED=1 selects the fused single pass (gp_fused_pass) when
// the 4-slot camera vector fits one CTA's shared memory; SSFM_FUSED=0 two-pass.
static int setup_gp_pcg_op(ssfm_handle* h, cudaStream_t st) {
  h->pcg_sms = pcg_sms_of(h);
  h->graph_state = -1;
  const int C = h->gp.gp.C;
  const char* env = getenv("SSFM_FUSED");
  const bool want = env ? env[0] != '0' : false;
  if (want && C < FZ_MAX_CAMERAS) {
    cudaFuncAttributes fa;
    CU(cudaFuncGetAttributes(&fa, gp_k_pcg<true>));
    int optin = 0;
    CU(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device));
    const size_t dyn = sizeof(double) * (4ull * C + FZ_WARPS * 32 * 4) + sizeof(int) * (size_t)C;
    int occ = 0;
    if (fa.sharedSizeBytes + dyn <= (size_t)optin) {
      CU(cudaFuncSetAttribute(gp_k_pcg<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
      CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gp_k_pcg<true>, FZ_THREADS, dyn));
    }
    if (occ >= 1) {
      h->pcg_grid = occ * h->pcg_sms;
      h->pcg_threads = FZ_THREADS;
      h->pcg_smem = dyn;
      h->pcg_fn = (void*)gp_k_pcg<true>;
      h->fz.G = 1;
      h->fz.SL = 4;
      h->fz.ngrp = h->pcg_grid;
      int ok = 0, rc;
      if ((rc = build_fused_schedule(h, 4, h->gp.status, st, &ok))) return rc;
      if (ok) return SSFM_OK;
    }
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gp_k_pcg<false>, PCG_THREADS, 0) || occ < 1)
    return set_err(SSFM_CUDA_ERROR, "occupancy query for the PCG kernel failed");
  h->pcg_grid = occ * h->pcg_sms;
  h->pcg_threads = PCG_THREADS;
  h->pcg_smem = 0;
  h->pcg_fn = (void*)gp_k_pcg<false>;
  h->fz = FusedTopo{};
  // the two-pass GP operator runs as a CUDA graph (gp_pcg_graph.cuh) from
  // 250k observations on single-rank handles; SSFM_GP_GRAPH=1 / 0 forces either
  const char* ge = getenv("SSFM_GP_GRAPH");
  h->graph_state = (ge ? ge[0] == '1' : h->topo.N >= 250000) ? 0 : -1;
  return SSFM_OK;
}


static int setup_ba_pcg(ssfm_handle* h, cudaStream_t st) {
  int rc = setup_ba_pcg_op(h, st);
  if (rc) return rc;
  // two-pass operator: the camera pass reads factored records (ba_factor,
  // 7 / 9 doubles per observation instead of 16; SSFM_FACTORED=0: off)
  const char* fe = getenv("SSFM_FACTORED");
  if (h->fz.G == 0 && !(fe && fe[0] == '0')) {
    BADev& d = h->ba;
    DALLOC(d.Fcm, fcm_doubles(d.bp.model, d.Npad));
    DALLOC(d.camlin, d.bp.C);
    h->pcg_fn = (void*)ba_k_pcg<0, true>;
    // and the point pass the omega form (ba_wobs: Jp + Jf, 8 doubles per
    // observation instead of the 16-double record; SSFM_WFORM=0: off)
    const char* we = getenv("SSFM_WFORM");
    if (!(we && we[0] == '0')) {
      DALLOC(d.Gpm, 8ll * d.Npad);
      DALLOC(d.Xl, 4ll * d.bp.P);
      DALLOC(d.Wc, 8ll * d.bp.C);
      // linearize evaluates each observation once (ba_k_lin_tile +
      // ba_k_lin_points; SSFM_LIN2=0: the two evaluating passes)
      const char* le = getenv("SSFM_LIN2");
      if (!(le && le[0] == '0')) DALLOC(d.Rpm, 4ll * d.Npad);
    }
  }
  const char* ge = getenv("SSFM_PCG_GRAPH");
  // two-pass operator from 250k observations: the graph wins well below C5
  // (3000 cameras / 800k obs: 0.067 vs 0.116 ms per CG iteration)
  const bool want = ge ? ge[0] == '1' : (h->fz.G == 0 && h->topo.N >= 250000);
  h->graph_state = want ? 0 : -1;
  return SSFM_OK;
}

static int setup_ba_pcg_op(ssfm_handle* h, cudaStream_t st) {
  // SSFM_PCG_SMS caps the SMs of the persistent PCG grid (several sharded
  // handles on one device must be co-resident: their kernels wait on each other)
  h->pcg_sms = pcg_sms_of(h);
  const int C = h->ba.bp.C;
  const char* env = getenv("SSFM_FUSED");
  // Default: fused below 250k observations; from there the two-pass operator
  // with the factored camera pass in the CUDA graph is faster (C4-BA 4M obs:
  // 0.169 vs 0.21 ms per CG iteration; C3 680k: 0.056 vs 0.066).
  // SSFM_FUSED=1 (or 2/4/8) forces the fused operator, SSFM_FUSED=0 two-pass.
  const bool want = (env ? env[0] != '0' : h->topo.N < 250000) && C < FZ_MAX_CAMERAS;
  // SSFM_FUSED=0 forces the two-pass operator; SSFM_FUSED=2/4/8 forces that many
  // slot groups (tests exercise the multi-group path on small problems)
  const int force_g = (env && (env[0] == '2' || env[0] == '4' || env[0] == '8')) ? env[0] - '0' : 1;
  int ok = 0, rc;
  if (want && force_g <= 1 && (rc = try_fused_ba<8>(h, &ok))) return rc;
  // By default only the single-group fused operator is used: with G > 1 the
  // redundant point-side work of the G CTAs costs more than the second
  // Jacobian read it saves (measured at C5: 1.91 vs 1.32 ms per CG iteration).
  const bool multi = force_g > 1;
  if (want && multi && !ok && force_g <= 2 && (rc = try_fused_ba<4>(h, &ok))) return rc;
  if (want && multi && !ok && force_g <= 4 && (rc = try_fused_ba<2>(h, &ok))) return rc;
  if (want && multi && !ok && (rc = try_fused_ba<1>(h, &ok))) return rc;
  if (ok) {
    if ((rc = build_fused_schedule(h, 8, h->ba.status, st, &ok))) return rc;
    if (ok) return SSFM_OK;
  }
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ba_k_pcg<0>, PCG_THREADS, 0) || occ < 1)
    return set_err(SSFM_CUDA_ERROR, "occupancy query for the PCG kernel failed");
  h->pcg_grid = occ * h->pcg_sms;
  h->pcg_threads = PCG_THREADS;
  h->pcg_smem = 0;
  h->pcg_fn = (void*)ba_k_pcg<0>;
  h->fz = FusedTopo{};
  return SSFM_OK;
}

// ---------------------------------------------------------------------------
// BA
// ---------------------------------------------------------------------------
static int create_ba(const ssfm_ba_desc* desc, ssfm_arena* arena, void* stream, ssfm_handle** out);
static int create_gp(const ssfm_gp_desc* desc, ssfm_arena* arena, void* stream, ssfm_handle** out);

extern "C" int ssfm_create_ba(const ssfm_ba_desc* desc, void* stream, ssfm_handle** out) {
  return create_ba(desc, nullptr, stream, out);
}
extern "C" int ssfm_create_gp(const ssfm_gp_desc* desc, void* stream, ssfm_handle** out) {
  return create_gp(desc, nullptr, stream, out);
}
extern "C" int ssfm_create_ba_in(const ssfm_ba_desc* desc, ssfm_arena* arena, void* stream, ssfm_handle** out) {
  if (!arena) return set_err(SSFM_INVALID_ARGUMENT, "null arena");
  return create_ba(desc, arena, stream, out);
}
extern "C" int ssfm_create_gp_in(const ssfm_gp_desc* desc, ssfm_arena* arena, void* stream, ssfm_handle** out) {
  if (!arena) return set_err(SSFM_INVALID_ARGUMENT, "null arena");
  return create_gp(desc, arena, stream, out);
}

extern "C" int ssfm_arena_create(int32_t device, int64_t reserve_bytes, ssfm_arena** out) {
  if (!out || reserve_bytes < 0) return set_err(SSFM_INVALID_ARGUMENT, "bad argument");
  int cur = 0;
  CU(cudaGetDevice(&cur));
  ssfm_arena* a = new ssfm_arena();
  a->device = device < 0 ? cur : device;
  if (a->device != cur) {
    delete a;
    return set_err(SSFM_INVALID_ARGUMENT, "arena device must be the current device");
  }
  if (reserve_bytes > 0) {
    char* p = nullptr;
    if (cudaMalloc((void**)&p, (size_t)reserve_bytes) != cudaSuccess) {
      cudaGetLastError();
      delete a;
      return set_err(SSFM_CUDA_ERROR, "arena: cudaMalloc of the reservation failed");
    }
    a->chunks.emplace_back(p, (size_t)reserve_bytes);
    a->chunk_mallocs = 1;
  }
  *out = a;
  return SSFM_OK;
}

extern "C" int ssfm_arena_destroy(ssfm_arena* a) {
  if (!a) return SSFM_OK;
  {
    std::lock_guard<std::mutex> lk(a->mu);
    if (a->live > 0) return set_err(SSFM_INVALID_ARGUMENT, "arena still has live handles");
  }
  cudaDeviceSynchronize();
  for (auto& c : a->chunks) cudaFree(c.first);
  delete a;
  return SSFM_OK;
}

extern "C" int ssfm_arena_info(ssfm_arena* a, int64_t* capacity, int64_t* high_water, int32_t* live_handles,
                               int64_t* chunk_mallocs) {
  if (!a) return set_err(SSFM_INVALID_ARGUMENT, "null arena");
  std::lock_guard<std::mutex> lk(a->mu);
  if (capacity) *capacity = (int64_t)arena_capacity(a);
  if (high_water) *high_water = (int64_t)a->high_water;
  if (live_handles) *live_handles = a->live;
  if (chunk_mallocs) *chunk_mallocs = a->chunk_mallocs;
  return SSFM_OK;
}

static int create_ba(const ssfm_ba_desc* desc, ssfm_arena* arena, void* stream, ssfm_handle** out) {
  if (!desc || !out) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (desc->num_obs <= 0) return set_err(SSFM_EMPTY_PROBLEM, "scene has no observations");
  if (desc->num_obs >= (1ll << 31) - 64) return set_err(SSFM_INVALID_ARGUMENT, "too many observations for int32 indexing");
  if (desc->num_cameras <= 0 || desc->num_points < 0) return set_err(SSFM_INVALID_ARGUMENT, "bad camera/point counts");
  cudaStream_t st = (cudaStream_t)stream;
  ssfm_handle* h = new ssfm_handle();
  CU(cudaGetDevice(&h->device));
  CU(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device));
  h->kind = 0;
  if (arena) {
    if (arena->device != h->device) { delete h; return set_err(SSFM_INVALID_ARGUMENT, "arena is on another device"); }
    std::lock_guard<std::mutex> lk(arena->mu);
    arena->live++;
    h->arena = arena;
  }
  const int C = desc->num_cameras, P = desc->num_points;
  const long long N = desc->num_obs;
  BADev& d = h->ba;
  d.bp.C = C; d.bp.P = P; d.bp.N = N;
  d.bp.model = desc->model;
  d.bp.focal_mode = desc->optimize_focal ? (desc->shared_focal ? 2 : 1) : 0;
  if (desc->loss_kind < 0 || desc->loss_kind > 2) {
    free_handle(h);
    return set_err(SSFM_INVALID_ARGUMENT, "unknown loss kind");
  }
  d.bp.loss_kind = desc->loss_kind;
  d.bp.delta = desc->loss_delta;
  d.bp.off_pts = 7ll * C;
  d.bp.off_foc = 7ll * C + 3ll * P;
  h->total_params = 7ll * C + 3ll * P + (d.bp.focal_mode == 1 ? C : d.bp.focal_mode == 2 ? 1 : 0);
  h->total_res = 2 * N;
  auto fail = [&](int rc) { free_handle(h); return rc; };
  // SSFM_TIMING=1: phase times of the creation on stderr (diagnostic)
  const bool timing = getenv("SSFM_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!timing) return;
    cudaStreamSynchronize(st);
    auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[ssfm create] %s %.1f ms\n", what, std::chrono::duration<double, std::milli>(t - t_last).count());
    t_last = t;
  };
  int rc;
  int* dstatus;
  if ((rc = dalloc(h, &dstatus, 1))) return fail(rc);
  d.status = dstatus;
  if ((rc = build_topo(h, desc->cam_idx, desc->pt_idx, C, P, N, st, dstatus))) return fail(rc);
  mark("topology");
  d.topo = h->topo;
  const Topo& T = h->topo;
  d.Npad = (N + 31) & ~31ll;
  double *pix_pm, *pps, *dists, *focals;
  if ((rc = dalloc(h, &pix_pm, 2 * N))) return fail(rc);
  if ((rc = dalloc(h, &pps, 2 * C))) return fail(rc);
  if ((rc = dalloc(h, &dists, 2 * C))) return fail(rc);
  if ((rc = dalloc(h, &focals, C))) return fail(rc);
  k_gather_rows<<<nblk(N, 256), 256, 0, st>>>(desc->pixels, T.pm_obs, N, 2, pix_pm);
  double* pix_cm;
  if ((rc = dalloc(h, &pix_cm, 2 * N))) return fail(rc);
  k_gather_rows<<<nblk(N, 256), 256, 0, st>>>(desc->pixels, T.cm_obs, N, 2, pix_cm);
  d.pix_cm = pix_cm;
  if (cudaMemcpyAsync(pps, desc->pps, sizeof(double) * 2 * C, cudaMemcpyDeviceToDevice, st) ||
      cudaMemcpyAsync(dists, desc->dists, sizeof(double) * 2 * C, cudaMemcpyDeviceToDevice, st))
    return fail(set_err(SSFM_CUDA_ERROR, "copy camera intrinsics"));
  if (desc->focals) {
    if (cudaMemcpyAsync(focals, desc->focals, sizeof(double) * C, cudaMemcpyDeviceToDevice, st))
      return fail(set_err(SSFM_CUDA_ERROR, "copy focals"));
  } else if (cudaMemsetAsync(focals, 0, sizeof(double) * C, st)) {
    return fail(set_err(SSFM_CUDA_ERROR, "memset focals"));
  }
  d.pix_pm = pix_pm; d.pps = pps; d.dists = dists; d.focals = focals;
  if ((rc = dalloc(h, &d.cams, C))) return fail(rc);
  if ((rc = dalloc(h, &d.Cpt, 6ll * P))) return fail(rc);
  if ((rc = dalloc(h, &d.gpt, 3ll * P))) return fail(rc);
  if ((rc = dalloc(h, &d.Bc, 64ll * C))) return fail(rc);
  if ((rc = dalloc(h, &d.gcam, 8ll * C))) return fail(rc);
  if ((rc = dalloc(h, &d.tilebuf, (long long)CAM_V * T.nt))) return fail(rc);
  if ((rc = dalloc(h, &d.Cinv, 6ll * P))) return fail(rc);
  if ((rc = dalloc(h, &d.y0, 3ll * P))) return fail(rc);
  if ((rc = dalloc(h, &d.yv, 4ll * P))) return fail(rc);   // padded: 32-byte gathers
  if ((rc = dalloc(h, &d.Minv, 64ll * C))) return fail(rc);
  if ((rc = dalloc(h, &d.bred, 8ll * C))) return fail(rc);
  if ((rc = dalloc(h, &d.fterm, 2ll * C))) return fail(rc);
  d.fpt = nullptr;
  d.fwpart = nullptr;
  if (d.bp.focal_mode == 2) {
    if ((rc = dalloc(h, &d.fpt, 3ll * P))) return fail(rc);
    if ((rc = dalloc(h, &d.fwpart, nblk(P, 256) + 1))) return fail(rc);
  }
  if ((rc = dalloc(h, &d.pinned, C))) return fail(rc);
  if ((rc = common_alloc(h, 8 * C, C))) return fail(rc);
  d.scal = h->misc->scal;
  d.status = &h->misc->status;
  mark("arrays");
  // launch geometry of the PCG kernel (fused single-pass operator when the
  // camera vector fits the shared memory of <= 8 CTAs, else two-pass)
  if ((rc = setup_ba_pcg(h, st))) return fail(rc);
  // the camera-major Jacobian copy: only without the factored record (the
  // fused operator, SSFM_FACTORED=0); two-pass handles read Fcm instead
  if (!d.Fcm && (rc = dalloc(h, &d.Jcm, BA_JREC * d.Npad))) return fail(rc);
  // the point-major record: Jp + Jf for omega-form handles, else the full record
  if (!d.Gpm && (rc = dalloc(h, &d.Jpm, BA_JREC * d.Npad))) return fail(rc);
  mark("pcg setup");
  h->lin_blocks = std::max(1, std::min(nblk(T.nb, 8), h->num_sms * 16));
  h->cost_blocks = nblk(N, 256);
  h->cam_blocks = nblk(C, 256);
  h->red_n = std::max<long long>(std::max<long long>(h->cost_blocks, T.nt),
                                 (long long)h->lin_blocks * 8 + h->cam_blocks);
  if ((rc = dalloc(h, &h->red, h->red_n))) return fail(rc);
  if ((rc = dalloc(h, &h->part, 3ll * h->pcg_grid + 2))) return fail(rc);
  d.partials = h->red;
  if (cudaMemsetAsync(h->misc, 0, sizeof(Misc), st) || cudaStreamSynchronize(st))
    return fail(set_err(SSFM_CUDA_ERROR, "init"));
  if (cudaGetLastError() != cudaSuccess) return fail(set_err(SSFM_CUDA_ERROR, "setup kernel launch failed"));
  *out = h;
  return SSFM_OK;
}


// ---------------------------------------------------------------------------
// GP
// ---------------------------------------------------------------------------
static int create_gp(const ssfm_gp_desc* desc, ssfm_arena* arena, void* stream, ssfm_handle** out) {
  if (!desc || !out) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (desc->num_obs <= 0) return set_err(SSFM_EMPTY_PROBLEM, "problem has no observations");
  if (desc->num_obs >= (1ll << 31) - 64) return set_err(SSFM_INVALID_ARGUMENT, "too many observations for int32 indexing");
  if (desc->num_cameras <= 0 || desc->num_points < 0) return set_err(SSFM_INVALID_ARGUMENT, "bad camera/point counts");
  if (desc->depth_mode && !desc->depths) return set_err(SSFM_MISSING_DEPTH, "depth mode requires a depth per observation");
  cudaStream_t st = (cudaStream_t)stream;
  ssfm_handle* h = new ssfm_handle();
  CU(cudaGetDevice(&h->device));
  CU(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device));
  h->kind = 1;
  if (arena) {
    if (arena->device != h->device) { delete h; return set_err(SSFM_INVALID_ARGUMENT, "arena is on another device"); }
    std::lock_guard<std::mutex> lk(arena->mu);
    arena->live++;
    h->arena = arena;
  }
  const int C = desc->num_cameras, P = desc->num_points;
  const long long N = desc->num_obs;
  GPDev& g = h->gp;
  g.gp.C = C; g.gp.P = P; g.gp.N = N;
  g.gp.depth_mode = desc->depth_mode;
  g.gp.gauge_fixed = desc->gauge_fixed;
  if (desc->loss_kind < 0 || desc->loss_kind > 2) {
    free_handle(h);
    return set_err(SSFM_INVALID_ARGUMENT, "unknown loss kind");
  }
  g.gp.loss_kind = desc->loss_kind;
  g.gp.delta = desc->loss_delta;
  g.gp.off_pts = 3ll * C;
  g.gp.off_sc = 3ll * C + 3ll * P;
  h->total_params = 3ll * C + 3ll * P + (desc->depth_mode ? 0 : N);
  h->total_res = 3 * N;
  auto fail = [&](int rc) { free_handle(h); return rc; };
  int rc;
  int* dstatus;
  if ((rc = dalloc(h, &dstatus, 1))) return fail(rc);
  if ((rc = build_topo(h, desc->cam_idx, desc->pt_idx, C, P, N, st, dstatus))) return fail(rc);
  g.topo = h->topo;
  const Topo& T = h->topo;
  g.Npad = (N + 31) & ~31ll;
  double *ray_pm, *dep_pm = nullptr;
  if ((rc = dalloc(h, &ray_pm, 3 * N))) return fail(rc);
  k_gather_rows<<<nblk(N, 256), 256, 0, st>>>(desc->rays, T.pm_obs, N, 3, ray_pm);
  if (desc->depth_mode) {
    if ((rc = dalloc(h, &dep_pm, N))) return fail(rc);
    k_gather_rows<<<nblk(N, 256), 256, 0, st>>>(desc->depths, T.pm_obs, N, 1, dep_pm);
  }
  g.ray_pm = ray_pm; g.dep_pm = dep_pm;
  double *ray_cm, *dep_cm = nullptr;
  if ((rc = dalloc(h, &ray_cm, 3 * N))) return fail(rc);
  k_gather_rows<<<nblk(N, 256), 256, 0, st>>>(desc->rays, T.cm_obs, N, 3, ray_cm);
  if (desc->depth_mode) {
    if ((rc = dalloc(h, &dep_cm, N))) return fail(rc);
    k_gather_rows<<<nblk(N, 256), 256, 0, st>>>(desc->depths, T.cm_obs, N, 1, dep_cm);
  }
  g.ray_cm = ray_cm; g.dep_cm = dep_cm;
  if ((rc = dalloc(h, &g.Jpm, GP_JREC * g.Npad))) return fail(rc);
  if ((rc = dalloc(h, &g.Jcm, GP_JREC * g.Npad))) return fail(rc);
  if ((rc = dalloc(h, &g.rcm, 3 * g.Npad))) return fail(rc);
  if ((rc = dalloc(h, &g.bo_pm, N))) return fail(rc);
  if ((rc = dalloc(h, &g.bo_cm, N))) return fail(rc);
  if ((rc = dalloc(h, &g.gsc, N))) return fail(rc);
  if ((rc = dalloc(h, &g.Apt, P))) return fail(rc);
  if ((rc = dalloc(h, &g.gpt, 3ll * P))) return fail(rc);
  if ((rc = dalloc(h, &g.Acam, C))) return fail(rc);
  if ((rc = dalloc(h, &g.gcam, 3ll * C))) return fail(rc);
  if ((rc = dalloc(h, &g.Minv_pt, 6ll * P))) return fail(rc);
  if ((rc = dalloc(h, &g.y0, 3ll * P))) return fail(rc);
  if ((rc = dalloc(h, &g.yv, 4ll * P))) return fail(rc);   // padded: 32-byte gathers
  if ((rc = dalloc(h, &g.Bp, 6ll * C))) return fail(rc);
  if ((rc = dalloc(h, &g.Minv, 16ll * C))) return fail(rc);
  if ((rc = dalloc(h, &g.bred, 4ll * C))) return fail(rc);
  if ((rc = dalloc(h, &g.pinned, C))) return fail(rc);
  if ((rc = dalloc(h, &g.tilebuf, (long long)GPE_V * T.nt))) return fail(rc);
  if ((rc = common_alloc(h, 4 * C, C))) return fail(rc);
  g.scal = h->misc->scal;
  g.status = &h->misc->status;
  if ((rc = setup_gp_pcg_op(h, st))) return fail(rc);
  h->lin_blocks = std::max(1, std::min(nblk(T.nb, 8), h->num_sms * 16));
  h->cost_blocks = nblk(N, 256);
  h->cam_blocks = nblk(C, 256);
  h->red_n = std::max<long long>(h->cost_blocks, (long long)h->lin_blocks * 8 + h->cam_blocks + nblk(N, 256));
  if ((rc = dalloc(h, &h->red, h->red_n))) return fail(rc);
  if ((rc = dalloc(h, &h->part, 3ll * h->pcg_grid + 2))) return fail(rc);
  g.partials = h->red;
  if (cudaMemsetAsync(h->misc, 0, sizeof(Misc), st) || cudaStreamSynchronize(st))
    return fail(set_err(SSFM_CUDA_ERROR, "init"));
  if (cudaGetLastError() != cudaSuccess) return fail(set_err(SSFM_CUDA_ERROR, "setup kernel launch failed"));
  *out = h;
  return SSFM_OK;
}

// ---------------------------------------------------------------------------
// pattern export (JtJPattern.off_keys / _SchurPlan slots)
// ---------------------------------------------------------------------------
static int sort_unique(ssfm_handle* h, unsigned long long* codes, long long n, long long* n_out,
                       unsigned long long** uniq, std::vector<void*>& tmp_allocs, cudaStream_t st) {
  unsigned long long *sorted = nullptr, *un = nullptr;
  int* nsel = nullptr;
  CU(cudaMalloc(&sorted, sizeof(unsigned long long) * std::max(n, 1ll)));
  CU(cudaMalloc(&un, sizeof(unsigned long long) * std::max(n, 1ll)));
  CU(cudaMalloc(&nsel, sizeof(int)));
  tmp_allocs.push_back(sorted); tmp_allocs.push_back(un); tmp_allocs.push_back(nsel);
  size_t b1 = 0, b2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, b1, codes, sorted, (int)n, 0, 64, st);
  cub::DeviceSelect::Unique(nullptr, b2, sorted, un, nsel, (int)n, st);
  void* tmp = nullptr;
  CU(cudaMalloc(&tmp, std::max(b1, b2)));
  tmp_allocs.push_back(tmp);
  size_t bb = std::max(b1, b2);
  CU(cub::DeviceRadixSort::SortKeys(tmp, bb, codes, sorted, (int)n, 0, 64, st));
  bb = std::max(b1, b2);
  CU(cub::DeviceSelect::Unique(tmp, bb, sorted, un, nsel, (int)n, st));
  int hn = 0;
  CU(cudaMemcpyAsync(&hn, nsel, sizeof(int), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  *n_out = hn;
  *uniq = un;
  (void)h;
  return SSFM_OK;
}

static int export_keys(ssfm_handle* h, int32_t* off_keys, int64_t off_cap, int64_t* n_off,
                       int32_t* slots, int64_t slot_cap, int64_t* n_slots, cudaStream_t st) {
  const Topo& T = h->topo;
  const int kind = h->kind;
  const int C = T.C, P = T.P;
  const long long N = T.N;
  int F = 0, nscale = 0;
  long long nblocks;
  // focal code for the pattern kernels: 2 per-camera, 1 shared, 0 none
  const int Fr = (kind == 0) ? (h->ba.bp.focal_mode == 1 ? 2 : h->ba.bp.focal_mode == 2 ? 1 : 0) : 0;
  if (kind == 0) {
    F = h->ba.bp.focal_mode == 1 ? C : h->ba.bp.focal_mode == 2 ? 1 : 0;
    nblocks = (long long)C + P + F;
  } else {
    nscale = h->gp.gp.depth_mode ? 0 : (int)N;
    nblocks = (long long)C + P + nscale;
  }
  std::vector<void*> tmp;
  int rc = SSFM_OK;
  if (off_keys || n_off) {
    const int per = (kind == 0) ? (F ? 3 : 1) : (nscale ? 3 : 1);
    unsigned long long* codes = nullptr;
    if (cudaMalloc(&codes, sizeof(unsigned long long) * per * N)) rc = set_err(SSFM_CUDA_ERROR, "alloc");
    else {
      tmp.push_back(codes);
      k_offkey_codes<<<nblk(N, 256), 256, 0, st>>>(T.pm_cam, T.pm_pt, T.pm_obs, N, kind, C, P,
                                                   Fr, nscale, nblocks, codes);
      long long K = 0;
      unsigned long long* un = nullptr;
      rc = sort_unique(h, codes, per * N, &K, &un, tmp, st);
      if (!rc) {
        if (n_off) *n_off = K;
        if (off_keys && off_cap >= K && K > 0)
          k_decode_pairs<<<nblk(K, 256), 256, 0, st>>>(un, K, nblocks, off_keys);
      }
    }
  }
  if (!rc && (slots || n_slots)) {
    long long *cnt = nullptr, *off = nullptr;
    if (cudaMalloc(&cnt, sizeof(long long) * (P + 1)) || cudaMalloc(&off, sizeof(long long) * (P + 1)))
      rc = set_err(SSFM_CUDA_ERROR, "alloc");
    else {
      tmp.push_back(cnt); tmp.push_back(off);
      cudaMemsetAsync(cnt, 0, sizeof(long long) * (P + 1), st);
      if (P) k_slot_count<<<nblk(P, 256), 256, 0, st>>>(T.pt_seg, P, kind, Fr, cnt);
      size_t bb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, bb, cnt, off, P + 1, st);
      void* t2 = nullptr;
      cudaMalloc(&t2, bb);
      tmp.push_back(t2);
      cub::DeviceScan::ExclusiveSum(t2, bb, cnt, off, P + 1, st);
      long long total = 0;
      cudaMemcpyAsync(&total, off + P, sizeof(long long), cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      unsigned long long* codes = nullptr;
      if (cudaMalloc(&codes, sizeof(unsigned long long) * std::max(total, 1ll))) rc = set_err(SSFM_CUDA_ERROR, "alloc");
      else {
        tmp.push_back(codes);
        if (P) k_slot_codes<<<nblk(P, 256), 256, 0, st>>>(T.pt_seg, T.pm_cam, P, kind, C, Fr, off, codes);
        long long S = 0;
        unsigned long long* un = nullptr;
        rc = sort_unique(h, codes, total, &S, &un, tmp, st);
        if (!rc) {
          if (n_slots) *n_slots = S;
          const long long nret = (long long)C + (kind == 0 ? (Fr == 1 ? 1 : (Fr ? C : 0)) : 0);
          if (slots && slot_cap >= S && S > 0)
            k_decode_pairs<<<nblk(S, 256), 256, 0, st>>>(un, S, nret, slots);
        }
      }
    }
  }
  cudaStreamSynchronize(st);
  for (void* p : tmp) cudaFree(p);
  if (!rc && cudaGetLastError() != cudaSuccess) rc = set_err(SSFM_CUDA_ERROR, "pattern export kernel failed");
  return rc;
}

// ---------------------------------------------------------------------------
// generic dispatch helpers
// ---------------------------------------------------------------------------
static void count_launch(ssfm_handle* h, int n = 1) { h->prof.kernel_launches += n; }

static bool sharded(const ssfm_handle* h) { return h->cm.nranks > 1; }

// peer-memory allreduce of n doubles in place (comm.cuh), stream-ordered
static int allreduce(ssfm_handle* h, double* data, long long n, int op, cudaStream_t st) {
  if (!sharded(h) || n <= 0) return SSFM_OK;
  if (n > h->cm.cap) return set_err(SSFM_INVALID_ARGUMENT, "allreduce larger than the exchange buffer");
  const int blocks = std::max(1, std::min(nblk(n, 256), h->num_sms));
  k_ar_post<<<blocks, 256, 0, st>>>(h->cm, data, n);
  k_ar_barrier<<<1, 32, 0, st>>>(h->cm);
  k_ar_reduce<<<blocks, 256, 0, st>>>(h->cm, data, n, op);
  count_launch(h, 3);
  CU(cudaGetLastError());
  return SSFM_OK;
}

// OR of the device status words over ranks (rejections must agree everywhere)
static int sync_status(ssfm_handle* h, cudaStream_t st) {
  if (!sharded(h)) return SSFM_OK;
  k_status_to_double<<<1, 1, 0, st>>>(&h->misc->status, h->ar_tmp);
  int rc = allreduce(h, h->ar_tmp, 1, AR_OR, st);
  if (rc) return rc;
  k_double_to_status<<<1, 1, 0, st>>>(h->ar_tmp, &h->misc->status);
  count_launch(h, 2);
  return SSFM_OK;
}

__global__ void k_add2(const double* a, const double* b, double* out) { *out = *a + *b; }

// cost(theta) -> misc.scal[SC_COST] (async)
static int launch_cost(ssfm_handle* h, const double* theta, cudaStream_t st) {
  if (h->kind == 0) {
    BADev& d = h->ba;
    ba_k_prep<<<h->cam_blocks, 256, 0, st>>>(d, theta);
    if (d.topo.nt) {   // camera tiles: the tile's camera is uniform (no per-observation camera gather)
      ba_k_cost_tile<<<d.topo.nt, SSFM_TILE, 0, st>>>(d, theta, h->red);
      k_sum_partials<<<1, 1024, 0, st>>>(h->red, d.topo.nt, d.scal + SC_COST);
    } else {
      ba_k_cost<<<h->cost_blocks, 256, 0, st>>>(d, theta, h->red);
      k_sum_partials<<<1, 1024, 0, st>>>(h->red, h->cost_blocks, d.scal + SC_COST);
    }
    count_launch(h, 3);
    int rc = allreduce(h, d.scal + SC_COST, 1, AR_SUM, st);
    if (rc) return rc;
  } else {
    GPDev& g = h->gp;
    gp_k_cost<<<h->cost_blocks, 256, 0, st>>>(g, theta, h->red);
    k_sum_partials<<<1, 1024, 0, st>>>(h->red, h->cost_blocks, g.scal + SC_COST);
    count_launch(h, 2);
    int rc = allreduce(h, g.scal + SC_COST, 1, AR_SUM, st);
    if (rc) return rc;
  }
  CU(cudaGetLastError());
  return SSFM_OK;
}

// linearize(theta) on device (async); grad max / norm into misc.scal
static int launch_linearize(ssfm_handle* h, const double* theta, double* r_out, double* J_out,
                            cudaStream_t st) {
  CU(zero_async(h->misc->scal + SC_GMAX, sizeof(double), st));
  if (h->kind == 0) {
    BADev& d = h->ba;
    ba_k_prep<<<h->cam_blocks, 256, 0, st>>>(d, theta);
    if (d.camlin) CU(copy_async(reinterpret_cast<double*>(d.camlin), reinterpret_cast<const double*>(d.cams),
                                (long long)(sizeof(BACam) / 8) * d.bp.C, st));
    if (d.Rpm && !r_out && !J_out) {   // each observation evaluated once (camera tiles), then point sums
      if (d.topo.nt) ba_k_lin_tile<<<d.topo.ng, SSFM_TILE, 0, st>>>(d, theta);   // tile groups
      ba_k_lin_points<<<h->lin_blocks, 256, 0, st>>>(d, theta, h->red);
    } else {
      ba_k_linearize<<<h->lin_blocks, 256, 0, st>>>(d, theta, r_out, J_out, h->red);
      if (d.topo.nt) ba_k_linearize_cm<<<d.topo.nt, SSFM_TILE, 0, st>>>(d, theta);
    }
    if (!sharded(h)) {
      ba_k_camfin<<<h->cam_blocks, 256, 0, st>>>(d, h->red + (long long)h->lin_blocks * 8, nullptr);
      k_sum_partials<<<1, 1024, 0, st>>>(h->red, h->lin_blocks * 8 + h->cam_blocks, d.scal + SC_GNORM2);
      count_launch(h, 5);
      if (d.bp.focal_mode == 2) { ba_k_shared_focal_grad<<<1, 256, 0, st>>>(d); count_launch(h); }
    } else {
      // camera blocks: local tile sums -> exchange -> identical Bc / gcam on every rank;
      // |g|^2 = sum over ranks of the point part + the (replicated) camera part
      k_cam_tilesum<<<h->cam_blocks, 256, 0, st>>>(d.topo, d.tilebuf, CAM_V, h->camsum);
      int rc = allreduce(h, h->camsum, (long long)CAM_V * d.bp.C, AR_SUM, st);
      if (rc) return rc;
      ba_k_camfin<<<h->cam_blocks, 256, 0, st>>>(d, h->red + (long long)h->lin_blocks * 8, h->camsum);
      k_sum_partials<<<1, 1024, 0, st>>>(h->red, h->lin_blocks * 8, h->ar_tmp + 1);
      if ((rc = allreduce(h, h->ar_tmp + 1, 1, AR_SUM, st))) return rc;
      k_sum_partials<<<1, 1024, 0, st>>>(h->red + (long long)h->lin_blocks * 8, h->cam_blocks, h->ar_tmp + 2);
      k_add2<<<1, 1, 0, st>>>(h->ar_tmp + 1, h->ar_tmp + 2, d.scal + SC_GNORM2);
      // shared focal: its gradient from the (replicated) camera sums
      if (d.bp.focal_mode == 2) { ba_k_shared_focal_grad<<<1, 256, 0, st>>>(d); count_launch(h); }
      if ((rc = allreduce(h, d.scal + SC_GMAX, 1, AR_MAX, st))) return rc;
      count_launch(h, 8);
    }
  } else {
    GPDev& g = h->gp;
    if (!sharded(h)) {
      int rc = gp_launch_linearize(g, theta, r_out, J_out, h->red, h->lin_blocks, h->cam_blocks, st);
      if (rc) return set_err(SSFM_CUDA_ERROR, "gp linearize launch");
      count_launch(h, 5);
    } else {
      // camera sums exchanged; |g|^2 = (points + scales: summed over ranks) + cameras
      gp_k_linearize<<<h->lin_blocks, 256, 0, st>>>(g, theta, r_out, J_out, h->red);
      if (g.topo.nt) gp_k_linearize_cm<<<g.topo.nt, SSFM_TILE, 0, st>>>(g, theta);
      k_cam_tilesum<<<h->cam_blocks, 256, 0, st>>>(g.topo, g.tilebuf, GPC_V, h->camsum);
      int rc = allreduce(h, h->camsum, (long long)GPC_V * g.gp.C, AR_SUM, st);
      if (rc) return rc;
      const long long off = (long long)h->lin_blocks * 8;
      gp_k_camfin<<<h->cam_blocks, 256, 0, st>>>(g, h->red + off, h->camsum);
      const int sb = nblk(g.topo.N, 256);
      gp_k_scale_norm<<<sb, 256, 0, st>>>(g, h->red + off + h->cam_blocks);
      k_sum_partials<<<1, 1024, 0, st>>>(h->red, (int)off, h->ar_tmp + 1);
      k_sum_partials<<<1, 1024, 0, st>>>(h->red + off + h->cam_blocks, sb, h->ar_tmp + 3);
      k_add2<<<1, 1, 0, st>>>(h->ar_tmp + 1, h->ar_tmp + 3, h->ar_tmp + 1);
      if ((rc = allreduce(h, h->ar_tmp + 1, 1, AR_SUM, st))) return rc;
      k_sum_partials<<<1, 1024, 0, st>>>(h->red + off, h->cam_blocks, h->ar_tmp + 2);
      k_add2<<<1, 1, 0, st>>>(h->ar_tmp + 1, h->ar_tmp + 2, g.scal + SC_GNORM2);
      if ((rc = allreduce(h, g.scal + SC_GMAX, 1, AR_MAX, st))) return rc;
      count_launch(h, 11);
    }
  }
  CU(cudaGetLastError());
  h->linearized = true;
  return SSFM_OK;
}


__global__ void k_g_setparams(CGGraphDev g, double lam, double cg_tol, int max_iters) {
  g.sc[0] = lam; g.sc[1] = cg_tol; g.ic[0] = max_iters; g.ic[4] = 0;
}

template <int SL>
static cudaError_t prepare_fused() {
  int optin = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, k_g_fused<SL>);
  if (e) return e;
  return cudaFuncSetAttribute(k_g_fused<SL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              optin - (int)fa.sharedSizeBytes);
}

template <int SL>
static void capture_fused(ssfm_handle* h, cudaStream_t cs) {
  k_g_fused<SL><<<h->pcg_grid, FZ_THREADS, h->pcg_smem, cs>>>(h->ba, h->fz, h->gdev);
}

// Keep a gathered per-point vector (y of the two-pass operator, 4P doubles)
// resident in L2 while the Jacobian streams past it: a persisting
// access-policy window on the stream the PCG graph is captured on (kernel
// nodes inherit it). Without it ~40 % of the camera pass's y gathers miss L2
// at C5 (0.39 GB of extra DRAM reads per CG iteration, ncu). SSFM_L2_PERSIST=0
// disables it. Returns whether the window was set.
static bool set_l2_window(ssfm_handle* h, cudaStream_t cs, void* base, size_t bytes) {
  const char* e = getenv("SSFM_L2_PERSIST");
  if (e && atoi(e) == 0) return false;
  int maxp = 0, maxw = 0;
  if (cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, h->device) != cudaSuccess ||
      cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, h->device) != cudaSuccess ||
      maxp <= 0 || maxw <= 0) {
    cudaGetLastError();
    return false;
  }
  const size_t win = std::min(bytes, (size_t)maxw);
  const size_t want = std::min(win, (size_t)maxp);
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
  if (cur < want && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaStreamAttrValue v = {};
  v.accessPolicyWindow.base_ptr = base;
  v.accessPolicyWindow.num_bytes = win;
  v.accessPolicyWindow.hitRatio = std::min(1.0f, (float)((double)want / (double)win));
  v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  if (cudaStreamSetAttribute(cs, cudaStreamAttributeAccessPolicyWindow, &v) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return true;
}

static void clear_l2_window(cudaStream_t cs) {
  cudaStreamAttrValue v = {};
  v.accessPolicyWindow.num_bytes = 0;
  cudaStreamSetAttribute(cs, cudaStreamAttributeAccessPolicyWindow, &v);
  cudaGetLastError();
}

// device state of the graph PCG (allocated once per handle)
static int alloc_gdev(ssfm_handle* h) {
  CGGraphDev& g = h->gdev;
  if (g.partA) return SSFM_OK;
  g.x = h->x; g.r = h->r; g.z = h->z; g.p = h->p; g.q = h->q;
  DALLOC(g.partA, 2 * CGV_BLOCKS + 2);
  DALLOC(g.partB, 2 * CGV_BLOCKS + 2);
  DALLOC(g.sc, 8);
  DALLOC(g.ic, 8);
  g.ctl = &h->misc->ctl;
  g.fused = (h->kind == 0 && h->fz.G > 0) ? 1 : 0;
  g.ngrp = h->kind == 0 ? h->fz.ngrp : 0;
  return SSFM_OK;
}

// one CG iteration of the BA graph PCG (the WHILE body), captured on cs;
// hc is the WHILE node's condition (set by k_g_scalars)
static void capture_ba_pcg_body(ssfm_handle* h, cudaStream_t cs, cudaGraphConditionalHandle hc) {
  CGGraphDev& g = h->gdev;
  BADev& d = h->ba;
  int occ_p = 0, occ_c = 0;
  const bool fac = d.Fcm != nullptr;
  void* kp = (void*)k_g_point;
  void* kc = fac ? (void*)k_g_camera<true> : (void*)k_g_camera<false>;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_p, kp, PTP_THREADS, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, kc, PCG_THREADS, 0);
  if (g.fused) {
    switch (h->fz.SL) {
      case 8: capture_fused<8>(h, cs); break;
      case 4: capture_fused<4>(h, cs); break;
      case 2: capture_fused<2>(h, cs); break;
      default: capture_fused<1>(h, cs); break;
    }
  } else {
    // SSFM_PTP_GRID_DIV (tests): a smaller point-pass grid (another batch partition; the
    // result must not depend on it)
    const char* gd = getenv("SSFM_PTP_GRID_DIV");
    const int div = gd ? std::max(1, atoi(gd)) : 1;
    k_g_point<<<std::max(1, std::max(1, occ_p) * h->num_sms / div), PTP_THREADS, 0, cs>>>(d, g);
    if (d.topo.nt) {
      if (fac) k_g_camera<true><<<std::max(1, occ_c) * h->num_sms, PCG_THREADS, 0, cs>>>(d, g);
      else k_g_camera<false><<<std::max(1, occ_c) * h->num_sms, PCG_THREADS, 0, cs>>>(d, g);
    }
  }
  if (sharded(h)) {   // exchange of the camera half of S*p between the passes and q
    k_gx_post<<<CGV_BLOCKS, 256, 0, cs>>>(d, h->fz, g, h->cm);
    k_gx_barrier<<<1, 32, 0, cs>>>(g, h->cm);
  }
  // the vector phases: one thread-block cluster kernel (k_g_vec), or four
  // grid-wide kernels (SSFM_GVEC=0)
  const char* gv = getenv("SSFM_GVEC");
  const bool cluster = !(gv && gv[0] == '0');
  if (cluster) {
    k_g_vec<<<GV_CL, GV_THREADS, 0, cs>>>(d, h->fz, g, h->cm, hc);
  } else {
    k_g_q<<<CGV_BLOCKS, 256, 0, cs>>>(d, h->fz, g, h->cm);
    k_g_update<<<CGV_BLOCKS, 256, 0, cs>>>(d, g, CGV_BLOCKS);
    k_g_pupdate<<<CGV_BLOCKS, 256, 0, cs>>>(d, g, CGV_BLOCKS);
    k_g_scalars<<<1, 32, 0, cs>>>(d, g, CGV_BLOCKS, hc);
  }
  h->graph_body_kernels = (g.fused ? 1 : 2) + (sharded(h) ? 2 : 0) + (cluster ? 1 : 4);
}

static cudaError_t prepare_fused_of(const ssfm_handle* h) {
  switch (h->fz.SL) {
    case 8: return prepare_fused<8>();
    case 4: return prepare_fused<4>();
    case 2: return prepare_fused<2>();
    default: return prepare_fused<1>();
  }
}

// Build the graph PCG of a BA handle: one conditional WHILE node, body = one
// CG iteration as kernels. Falls back to the persistent kernel (state -1) if
// the runtime refuses (e.g. no conditional nodes).
static int build_pcg_graph(ssfm_handle* h) {
  int rc = alloc_gdev(h);
  if (rc) return rc;
  CGGraphDev& g = h->gdev;
  cudaGraphConditionalHandle hc;
  cudaGraphNodeParams cp = {};
  cudaGraphNode_t cn;
  cudaStream_t cs = nullptr;
  auto unavailable = [&](cudaError_t e) {
    cudaGetLastError();
    if (cs) cudaStreamDestroy(cs);
    h->pcg_graph = nullptr;   // left to the driver: a half-captured body is not destroyed here
    h->graph_state = -1;
    (void)e;
    return SSFM_OK;
  };
  cudaError_t e;
  if (g.fused && (e = prepare_fused_of(h))) return unavailable(e);   // not while capturing
  if ((e = cudaGraphCreate(&h->pcg_graph, 0))) return unavailable(e);
  if ((e = cudaGraphConditionalHandleCreate(&hc, h->pcg_graph, 1, cudaGraphCondAssignDefault))) return unavailable(e);
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  if ((e = cudaGraphAddNode(&cn, h->pcg_graph, nullptr, 0, &cp))) return unavailable(e);
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking))) return unavailable(e);
  if (!g.fused) set_l2_window(h, cs, h->ba.yv, sizeof(double) * 4 * (size_t)h->ba.bp.P);
  if ((e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)))
    return unavailable(e);
  capture_ba_pcg_body(h, cs, hc);
  if ((e = cudaStreamEndCapture(cs, &body))) return unavailable(e);
  if ((e = cudaGraphInstantiate(&h->pcg_exec, h->pcg_graph, 0))) return unavailable(e);
  cudaStreamDestroy(cs);
  h->graph_state = 1;
  return SSFM_OK;
}

// GP: the PCG as a CUDA graph (gp_pcg_graph.cuh); single-rank two-pass handles
// one CG iteration of the GP graph PCG (the WHILE body), captured on cs
static void capture_gp_pcg_body(ssfm_handle* h, cudaStream_t cs, cudaGraphConditionalHandle hc) {
  CGGraphDev& g = h->gdev;
  GPDev& d = h->gp;
  int occ_p = 0, occ_c = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_p, (const void*)k_gg_point, PCG_THREADS, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, (const void*)k_gg_camera, PCG_THREADS, 0);
  k_gg_point<<<std::max(1, occ_p) * h->num_sms, PCG_THREADS, 0, cs>>>(d, g);
  if (d.topo.nt) k_gg_camera<<<std::max(1, occ_c) * h->num_sms, PCG_THREADS, 0, cs>>>(d, g);
  const char* gv = getenv("SSFM_GVEC");
  const bool cluster = !(gv && gv[0] == '0');
  if (cluster) {   // the vector phases as one thread-block cluster kernel
    k_gg_vec<<<GV_CL, GV_THREADS, 0, cs>>>(d, g, hc);
  } else {
    k_gg_q<<<CGV_BLOCKS, 256, 0, cs>>>(d, g);
    k_gg_update<<<CGV_BLOCKS, 256, 0, cs>>>(d, g, CGV_BLOCKS);
    k_gg_pupdate<<<CGV_BLOCKS, 256, 0, cs>>>(d, g, CGV_BLOCKS);
    k_g_scalars<<<1, 32, 0, cs>>>(d, g, CGV_BLOCKS, hc);
  }
  h->graph_body_kernels = 2 + (cluster ? 1 : 4);
}

// GP: the PCG as a CUDA graph (gp_pcg_graph.cuh); single-rank two-pass handles
static int build_gp_pcg_graph(ssfm_handle* h) {
  int rc = alloc_gdev(h);
  if (rc) return rc;
  cudaGraphConditionalHandle hc;
  cudaGraphNodeParams cp = {};
  cudaGraphNode_t cn;
  cudaStream_t cs = nullptr;
  auto unavailable = [&](cudaError_t e) {
    cudaGetLastError();
    if (cs) cudaStreamDestroy(cs);
    h->pcg_graph = nullptr;
    h->graph_state = -1;
    (void)e;
    return SSFM_OK;
  };
  cudaError_t e;
  if ((e = cudaGraphCreate(&h->pcg_graph, 0))) return unavailable(e);
  if ((e = cudaGraphConditionalHandleCreate(&hc, h->pcg_graph, 1, cudaGraphCondAssignDefault))) return unavailable(e);
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  if ((e = cudaGraphAddNode(&cn, h->pcg_graph, nullptr, 0, &cp))) return unavailable(e);
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking))) return unavailable(e);
  if ((e = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)))
    return unavailable(e);
  capture_gp_pcg_body(h, cs, hc);
  if ((e = cudaStreamEndCapture(cs, &body))) return unavailable(e);
  if ((e = cudaGraphInstantiate(&h->pcg_exec, h->pcg_graph, 0))) return unavailable(e);
  cudaStreamDestroy(cs);
  h->graph_state = 1;
  return SSFM_OK;
}

static int launch_pcg(ssfm_handle* h, double lam, const ssfm_lm_config* cfg, cudaStream_t st) {
  int max_it = cfg->cg_max_iters;
  double tol = cfg->cg_tol;
  // BA, one rank: the graph PCG for the two-pass operator on large problems,
  // where each pass as its own kernel (own occupancy, no grid barrier) beats
  // the persistent kernel (C5: 1.17 vs 1.29 ms per CG iteration); the
  // persistent kernel stays faster for the fused operator and small problems
  // (C4-BA fused 0.204 vs 0.229 ms, C1 0.025 vs 0.035 ms). SSFM_PCG_GRAPH=1/0
  // forces either.
  // (decided at handle creation, setup_ba_pcg; built here on first use)
  if (h->kind == 0 && h->graph_state == 1 && h->graph_sharded != sharded(h)) {
    // connected after the graph was built: rebuild it with the exchange kernels
    cudaGraphExecDestroy(h->pcg_exec);
    cudaGraphDestroy(h->pcg_graph);
    h->pcg_exec = nullptr;
    h->pcg_graph = nullptr;
    h->graph_state = 0;
  }
  if (h->kind == 1 && sharded(h)) h->graph_state = -1;   // sharded GP: persistent kernel (in-kernel exchange)
  if (h->kind == 1 && h->graph_state == 0) {
    int rc = build_gp_pcg_graph(h);
    if (rc) return rc;
  }
  if (h->kind == 1 && h->graph_state == 1) {
    CGGraphDev& g = h->gdev;
    k_g_setparams<<<1, 1, 0, st>>>(g, lam, tol, max_it);
    k_gg_init<<<CGV_BLOCKS, 256, 0, st>>>(h->gp, g);
    k_g_init2<<<1, 32, 0, st>>>(h->gp, g, CGV_BLOCKS);
    CU(cudaGraphLaunch(h->pcg_exec, st));
    count_launch(h, 3);
    h->graph_pending = true;
    return SSFM_OK;
  }
  if (h->kind == 0 && h->graph_state == 0) {
    const auto tg = std::chrono::steady_clock::now();
    int rc = build_pcg_graph(h);
    if (getenv("SSFM_TIMING"))
      fprintf(stderr, "[ssfm] graph build %.1f ms\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tg).count());
    if (rc) return rc;
    h->graph_sharded = sharded(h);
  }
  if (h->kind == 0 && h->graph_state == 1) {
    CGGraphDev& g = h->gdev;
    k_g_setparams<<<1, 1, 0, st>>>(g, lam, tol, max_it);
    k_g_init<<<CGV_BLOCKS, 256, 0, st>>>(h->ba, g);
    if (h->ba.Gpm) { k_cam_wvec<<<h->cam_blocks, 256, 0, st>>>(h->ba, g.p, h->ba.Wc); count_launch(h); }
    k_g_init2<<<1, 32, 0, st>>>(h->ba, g, CGV_BLOCKS);
    CU(cudaGraphLaunch(h->pcg_exec, st));
    count_launch(h, 3);
    h->graph_pending = true;   // the body kernels are counted once the CG count is known
    return SSFM_OK;
  }
  if (h->kind == 0) {
    BADev& d = h->ba;
    void* a[13];
    CGCtl* ctl = &h->misc->ctl;
    a[0] = &d; a[1] = &h->fz; a[2] = &h->cm; a[3] = &lam; a[4] = &max_it; a[5] = &tol;
    a[6] = &h->x; a[7] = &h->r; a[8] = &h->z; a[9] = &h->p; a[10] = &h->q;
    a[11] = &h->part; a[12] = &ctl;
    CU(cudaLaunchCooperativeKernel(h->pcg_fn, dim3(h->pcg_grid), dim3(h->pcg_threads), a, h->pcg_smem, st));
  } else {
    GPDev& g = h->gp;
    void* a[13];
    CGCtl* ctl = &h->misc->ctl;
    a[0] = &g; a[1] = &h->fz; a[2] = &h->cm; a[3] = &lam; a[4] = &max_it; a[5] = &tol;
    a[6] = &h->x; a[7] = &h->r; a[8] = &h->z; a[9] = &h->p; a[10] = &h->q;
    a[11] = &h->part; a[12] = &ctl;
    CU(cudaLaunchCooperativeKernel(h->pcg_fn, dim3(h->pcg_grid), dim3(h->pcg_threads), a, h->pcg_smem, st));
  }
  count_launch(h);
  return SSFM_OK;
}

// damped elimination blocks and the preconditioner at lambda (async)
static int launch_solve_pre(ssfm_handle* h, double lam, cudaStream_t st) {
  CU(zero_async(&h->misc->status, sizeof(int), st));
  CU(zero_async(&h->misc->ctl, sizeof(CGCtl), st));
  if (h->kind == 0) {
    BADev& d = h->ba;
    ba_k_ptinv<<<nblk(d.bp.P, 256), 256, 0, st>>>(d, lam);
    if (d.topo.nt) {
      if (d.Jcm) ba_k_precond<<<d.topo.nt, SSFM_TILE, 0, st>>>(d);
      else ba_k_precond_grp<<<d.topo.ng, SSFM_TILE, 0, st>>>(d);   // factored records: tile groups
    }
    const double* cs = nullptr;
    if (sharded(h)) {
      k_cam_tilesum<<<h->cam_blocks, 256, 0, st>>>(d.topo, d.tilebuf, CAM_V, h->camsum);
      int rc = allreduce(h, h->camsum, (long long)CAM_V * d.bp.C, AR_SUM, st);
      if (rc) return rc;
      cs = h->camsum;
      count_launch(h);
    }
    ba_k_camprec<<<nblk(d.bp.C, 64), 64, 0, st>>>(d, lam, cs);
    count_launch(h, 3);
    if (d.bp.focal_mode == 2) {
      const double* wsum = nullptr;
      if (sharded(h)) {   // sum_j a_j^T Cinv_j a_j over every rank's points
        k_sum_partials<<<1, 1024, 0, st>>>(d.fwpart, nblk(d.bp.P, 256), h->ar_tmp + 8);
        int rc = allreduce(h, h->ar_tmp + 8, 1, AR_SUM, st);
        if (rc) return rc;
        wsum = h->ar_tmp + 8;
        count_launch(h);
      }
      ba_k_shared_focal_prec<<<1, 256, 0, st>>>(d, nblk(d.bp.P, 256), wsum);
      count_launch(h);
    }
  } else {
    GPDev& g = h->gp;
    if (!sharded(h)) {
      int rc = gp_launch_elim(g, lam, h->cam_blocks, st);
      if (rc) return set_err(SSFM_CUDA_ERROR, "gp elimination launch");
      count_launch(h, 4);
    } else {
      g.lam = lam;
      const int lb = std::max(1, nblk(g.topo.nb, 8));
      gp_k_pt_elim<<<std::min(lb, 148 * 16), 256, 0, st>>>(g, lam);
      if (g.topo.nt) gp_k_cam_elim<<<g.topo.nt, SSFM_TILE, 0, st>>>(g, lam);
      k_cam_tilesum<<<h->cam_blocks, 256, 0, st>>>(g.topo, g.tilebuf, GPE_V, h->camsum);
      int rc = allreduce(h, h->camsum, (long long)GPE_V * g.gp.C, AR_SUM, st);
      if (rc) return rc;
      gp_k_camprec<<<nblk(g.gp.C, 64), 64, 0, st>>>(g, lam, h->camsum);
      count_launch(h, 4);
    }
  }
  CU(cudaGetLastError());
  return SSFM_OK;
}

// back-substitution of the PCG solution x -> delta (async)
static int launch_solve_post(ssfm_handle* h, cudaStream_t st) {
  if (h->kind == 0) {
    BADev& d = h->ba;
    if (d.Gpm) {   // omega form: the pipelined point pass with the W of x (ba_k_backsub_w)
      k_cam_wvec<<<h->cam_blocks, 256, 0, st>>>(d, h->x, d.Wc);
      count_launch(h);
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)ba_k_backsub_w, PTP_THREADS, 0);
      ba_k_backsub_w<<<std::max(1, occ) * h->num_sms, PTP_THREADS, 0, st>>>(d, h->delta);
    } else {
      ba_k_backsub<<<h->lin_blocks, 256, 0, st>>>(d, h->x, h->delta);
    }
    ba_k_camdelta<<<h->cam_blocks, 256, 0, st>>>(d, h->x, h->delta);
    count_launch(h, 2);
  } else {
    gp_launch_backsub(h->gp, h->x, h->delta, h->lin_blocks, h->cam_blocks, st);
    count_launch(h, 3);
  }
  CU(cudaGetLastError());
  return SSFM_OK;
}

// damped solve on the current linearization -> h->delta (async)
static int launch_solve(ssfm_handle* h, double lam, const ssfm_lm_config* cfg, cudaStream_t st) {
  int rc = launch_solve_pre(h, lam, st);
  if (rc) return rc;
  if (h->prof.on && !h->capturing) CU(cudaEventRecord(h->ev2, st));
  if ((rc = launch_pcg(h, lam, cfg, st))) return rc;
  if (h->prof.on && !h->capturing) CU(cudaEventRecord(h->ev3, st));
  return launch_solve_post(h, st);
}

static int launch_post_step(ssfm_handle* h, double* theta, cudaStream_t st) {
  if (h->kind == 0) {
    ba_k_renorm<<<h->cam_blocks, 256, 0, st>>>(h->ba.bp.C, theta, &h->misc->status);
    count_launch(h);
  } else {
    GPDev& g = h->gp;
    if (!sharded(h) || g.gp.depth_mode) {
      gp_launch_post_step(g, theta, h->red, st);
      count_launch(h, 3);
    } else {
      // mean scale over every rank's observations (gp.py:137-139)
      const int sb = nblk(g.topo.N, 256);
      gp_k_scale_sum<<<sb, 256, 0, st>>>(g, theta, h->red);
      gp_k_gauge_prep<<<1, 1024, 0, st>>>(g, h->red, sb, theta, h->ar_tmp + 4);
      int rc = allreduce(h, h->ar_tmp + 4, 2, AR_SUM, st);
      if (rc) return rc;
      gp_k_gauge_mean<<<1, 1, 0, st>>>(g, h->ar_tmp + 4);
      const long long n = g.gp.off_sc + g.topo.N;
      gp_k_gauge_apply<<<nblk(n, 256), 256, 0, st>>>(g, theta, n);
      count_launch(h, 4);
    }
  }
  CU(cudaGetLastError());
  return SSFM_OK;
}

static int read_misc(ssfm_handle* h, cudaStream_t st) {
  CU(cudaMemcpyAsync(h->hmisc, h->misc, sizeof(Misc), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  // a collective that timed out anywhere since the solve began (cost,
  // linearize, solve) leaves this rank's exchanged values invalid: fail loudly
  if (sharded(h) && (h->hmisc->status & ST_COMM_TIMEOUT))
    return set_err(SSFM_COMM_ERROR, "a peer rank did not reach the exchange in time (SSFM_COMM_TIMEOUT_S)");
  return SSFM_OK;
}

static int status_to_code(int s) {
  if (s & (ST_SINGULAR_POINT | ST_PIN_POINT | ST_SINGULAR_PRECOND | ST_PIN_RETAINED | ST_PIN_SCALE))
    return SSFM_SINGULAR_BLOCK;
  if (s & (ST_CG_MAXITER | ST_CG_BREAKDOWN)) return SSFM_CG_STALL;
  if (s & ST_ZERO_QUAT) return SSFM_ZERO_QUATERNION;
  if (s & (ST_COMM_TIMEOUT | ST_SCHEDULE)) return SSFM_COMM_ERROR;
  return SSFM_OK;
}

static std::string status_msg(int s, const Misc& m) {
  char buf[256];
  if (s & ST_SINGULAR_POINT) return "eliminable block singular after damping";
  if (s & ST_PIN_POINT) return "masked point direction with non-zero gradient";
  if (s & ST_PIN_SCALE) return "masked scale with non-zero coupling";
  if (s & ST_PIN_RETAINED) return "masked retained direction with non-zero gradient";
  if (s & ST_SINGULAR_PRECOND) return "singular preconditioner block";
  if (s & ST_CG_MAXITER) {
    snprintf(buf, sizeof buf, "CG did not reach tolerance in %d iterations (|r| %.3e, tol %.3e)",
             m.ctl.iters, m.ctl.rn, m.ctl.tol);
    return buf;
  }
  if (s & ST_CG_BREAKDOWN) return "CG broke down (p.q <= 0)";
  if (s & ST_ZERO_QUAT) return "quaternion norm below 1e-12 during renormalization";
  if (s & ST_COMM_TIMEOUT) return "a peer rank did not reach the exchange within 60 s";
  if (s & ST_SCHEDULE) return "fused operator schedule violated (internal error)";
  return "ok";
}

// ---------------------------------------------------------------------------
// public entry points
// ---------------------------------------------------------------------------
extern "C" const char* ssfm_last_error(void) { return g_last_error.c_str(); }
extern "C" const char* ssfm_version(void) { return "ssfm-b200 0.1 (sm_100a)"; }

extern "C" int ssfm_destroy(ssfm_handle* h) {
  free_handle(h);
  return SSFM_OK;
}

extern "C" int64_t ssfm_num_params(const ssfm_handle* h) { return h ? h->total_params : -1; }
extern "C" int64_t ssfm_num_residuals(const ssfm_handle* h) { return h ? h->total_res : -1; }
extern "C" int64_t ssfm_device_bytes(const ssfm_handle* h) { return h ? (int64_t)h->bytes : -1; }

extern "C" int ssfm_cost(ssfm_handle* h, const double* theta, double* cost_host, void* stream) {
  if (!h || !theta) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = launch_cost(h, theta, st);
  if (rc) return rc;
  if ((rc = read_misc(h, st))) return rc;
  if (cost_host) *cost_host = h->hmisc->scal[SC_COST];
  return SSFM_OK;
}

__global__ void k_export_grad_ba(BADev d, double* grad) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int C = d.bp.C, P = d.bp.P;
  if (i < 7ll * C) {
    grad[i] = d.gcam[8 * (i / 7) + (i % 7)];
  } else if (i < d.bp.off_foc) {
    grad[i] = d.gpt[i - 7ll * C];
  } else if (d.bp.focal_mode == 1 && i < d.bp.off_foc + C) {
    grad[i] = d.gcam[8 * (i - d.bp.off_foc) + 7];
  } else if (d.bp.focal_mode == 2 && i == d.bp.off_foc) {
    grad[i] = d.scal[SC_GFOCAL];
  }
  (void)P;
}

extern "C" int ssfm_linearize(ssfm_handle* h, const double* theta, double* r_out, double* J_out,
                              double* grad_out, double* grad_max_host, void* stream) {
  if (!h || !theta) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = launch_linearize(h, theta, r_out, J_out, st);
  if (rc) return rc;
  if (grad_out) {
    if (h->kind == 0) k_export_grad_ba<<<nblk(h->total_params, 256), 256, 0, st>>>(h->ba, grad_out);
    else gp_export_grad(h->gp, grad_out, st);
    CU(cudaGetLastError());
  }
  if ((rc = read_misc(h, st))) return rc;
  if (grad_max_host) *grad_max_host = h->hmisc->scal[SC_GMAX];
  return SSFM_OK;
}

extern "C" int ssfm_solve_normal(ssfm_handle* h, double lambda, const ssfm_lm_config* cfg,
                                 double* delta, int32_t* cg_iters_host, void* stream) {
  if (!h || !cfg) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  if (!h->linearized) return set_err(SSFM_INVALID_ARGUMENT, "ssfm_solve_normal before ssfm_linearize");
  if (lambda < 0) return set_err(SSFM_INVALID_ARGUMENT, "lambda must be non-negative");
  cudaStream_t st = (cudaStream_t)stream;
  int rc = launch_solve(h, lambda, cfg, st);
  if (rc) return rc;
  if (delta) CU(copy_async(delta, h->delta, h->total_params, st));
  if ((rc = sync_status(h, st))) return rc;
  if ((rc = read_misc(h, st))) return rc;
  const Misc& m = *h->hmisc;
  if (cg_iters_host) *cg_iters_host = m.ctl.iters;
  int code = status_to_code(m.status);
  if (code) return set_err(code, status_msg(m.status, m));
  return SSFM_OK;
}

extern "C" int ssfm_post_step(ssfm_handle* h, double* theta, void* stream) {
  if (!h || !theta) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  CU(zero_async(&h->misc->status, sizeof(int), st));
  int rc = launch_post_step(h, theta, st);
  if (rc) return rc;
  if ((rc = read_misc(h, st))) return rc;
  int code = status_to_code(h->hmisc->status);
  if (code) return set_err(code, status_msg(h->hmisc->status, *h->hmisc));
  return SSFM_OK;
}

// ---------------------------------------------------------------------------
// The LM loop as ONE CUDA graph (lm_graph.cuh): single-rank BA handles.
// ---------------------------------------------------------------------------
__global__ void k_g_setparams_lm(CGGraphDev g, const LMState* s, double cg_tol, int max_iters) {
  g.sc[0] = s->lam; g.sc[1] = cg_tol; g.ic[0] = max_iters; g.ic[4] = 0;
}
// the PCG WHILE node runs its body while the solve is not done (k_g_init2 decided)
__global__ void k_g_cond_init(CGGraphDev g, cudaGraphConditionalHandle hc) {
  cudaGraphSetConditional(hc, g.ic[3] ? 0u : 1u);
}
__global__ void k_lm_mark(LMState* s, int which) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  if (which == 0) s->t_pcg0 = t;
  else s->cg_pad_t1 = t;
}

// a conditional node at the capture position of st (its condition set by a
// kernel enqueued before it); the body graph is returned for capture
static cudaError_t cap_cond(cudaStream_t st, cudaGraphConditionalHandle hc, enum cudaGraphConditionalNodeType type,
                            cudaGraph_t* body) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  cudaError_t e = cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd);
  if (e) return e;
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = type;
  cp.conditional.size = 1;
  cudaGraphNode_t n;
  if ((e = cudaGraphAddNode(&n, g, deps, nd, &cp))) return e;
  if ((e = cudaStreamUpdateCaptureDependencies(st, &n, 1, cudaStreamSetCaptureDependencies))) return e;
  *body = cp.conditional.phGraph_out[0];
  return cudaSuccess;
}
static cudaError_t cap_handle(cudaStream_t st, cudaGraphConditionalHandle* hc) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g;
  cudaError_t e = cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, nullptr, nullptr);
  if (e) return e;
  return cudaGraphConditionalHandleCreate(hc, g, 0, 0);
}

static bool lm_graph_wanted(const ssfm_handle* h) {
  if (sharded(h) || h->lm_state < 0) return false;
  const char* e = getenv("SSFM_LM_GRAPH");
  return !(e && e[0] == '0');
}

static void destroy_lm_graph(ssfm_handle* h) {
  if (h->lm_exec) cudaGraphExecDestroy(h->lm_exec);
  if (h->lm_graph) cudaGraphDestroy(h->lm_graph);
  h->lm_exec = nullptr;
  h->lm_graph = nullptr;
  h->lm_state = 0;
}

static int build_lm_graph(ssfm_handle* h, const ssfm_lm_config* cfg) {
  const int cap = std::max(64, cfg->max_iterations);
  if (!h->lms) {
    DALLOC(h->lms, 1);
    CU(cudaMallocHost((void**)&h->hlms, sizeof(LMState)));
  }
  if (h->lrec_cap < cap) {
    DALLOC(h->lrecs, cap);   // handle-owned; an older smaller block stays with the handle
    if (h->hlrecs) cudaFreeHost(h->hlrecs);
    CU(cudaMallocHost((void**)&h->hlrecs, sizeof(LMRecDev) * cap));
    h->lrec_cap = cap;
  }
  const bool gpcg = h->graph_state != -1;   // the graph PCG (nested WHILE) or the persistent kernel
  if (gpcg) {
    int rc = alloc_gdev(h);
    if (rc) return rc;
  }
  const bool ba = h->kind == 0;
  double* scal = ba ? h->ba.scal : h->gp.scal;
  cudaStream_t s0 = nullptr, s1 = nullptr, s2 = nullptr;
  auto unavailable = [&](cudaError_t e) {
    cudaGetLastError();
    h->capturing = false;
    h->ba.lamp = nullptr;
    h->gp.lamp = nullptr;
    for (cudaStream_t x : {s0, s1, s2}) {
      if (!x) continue;
      cudaGraph_t junk = nullptr;
      cudaStreamCaptureStatus cst;
      if (cudaStreamIsCapturing(x, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone)
        cudaStreamEndCapture(x, &junk);
      cudaStreamDestroy(x);
    }
    cudaGetLastError();
    h->lm_graph = nullptr;
    h->lm_state = -1;
    if (getenv("SSFM_TIMING")) fprintf(stderr, "[ssfm] LM graph unavailable: %s\n", cudaGetErrorString(e));
    return SSFM_OK;
  };
  cudaError_t e;
  if (gpcg && h->gdev.fused && (e = prepare_fused_of(h))) return unavailable(e);
  for (cudaStream_t* x : {&s0, &s1, &s2})
    if ((e = cudaStreamCreateWithFlags(x, cudaStreamNonBlocking))) return unavailable(e);
  if ((e = cudaGraphCreate(&h->lm_graph, 0))) return unavailable(e);
  cudaGraphConditionalHandle hw, hlin, hsolve, hpcg;
  if ((e = cudaGraphConditionalHandleCreate(&hw, h->lm_graph, 1, cudaGraphCondAssignDefault))) return unavailable(e);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hw;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wn;
  if ((e = cudaGraphAddNode(&wn, h->lm_graph, nullptr, 0, &cp))) return unavailable(e);
  cudaGraph_t body = cp.conditional.phGraph_out[0], blin, bsolve, bpcg;
  BADev& d = h->ba;
  CGGraphDev& g = h->gdev;
  LMState* S = h->lms;
  const long long n = h->total_params;
  h->capturing = true;
  d.lamp = &S->lam;   // captured kernels read lambda from the loop state
  h->gp.lamp = &S->lam;
  const long long k0 = h->prof.kernel_launches;
  int rc = SSFM_OK;
  if ((e = cudaStreamBeginCaptureToGraph(s0, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)))
    return unavailable(e);
  if ((e = cap_handle(s0, &hlin))) return unavailable(e);
  k_lm_head<<<1, 1, 0, s0>>>(S, hlin);
  if ((e = cap_cond(s0, hlin, cudaGraphCondTypeIf, &blin))) return unavailable(e);
  // IF (need_lin): linearize + gradient test
  if ((e = cudaStreamBeginCaptureToGraph(s1, blin, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)))
    return unavailable(e);
  const long long k1 = h->prof.kernel_launches;
  if ((rc = launch_linearize(h, h->theta, nullptr, nullptr, s1))) { unavailable(cudaErrorUnknown); return rc; }
  k_lm_gradcheck<<<1, 1, 0, s1>>>(S, scal + SC_GMAX);
  h->lm_k_lin = h->prof.kernel_launches - k1 + 1;
  if ((e = cudaStreamEndCapture(s1, &blin))) return unavailable(e);
  if ((e = cap_handle(s0, &hsolve))) return unavailable(e);
  k_lm_mid<<<1, 1, 0, s0>>>(S, hsolve);
  if ((e = cap_cond(s0, hsolve, cudaGraphCondTypeIf, &bsolve))) return unavailable(e);
  // IF (not done): one damped solve, the candidate and the decision
  if ((e = cudaStreamBeginCaptureToGraph(s1, bsolve, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)))
    return unavailable(e);
  const long long k2 = h->prof.kernel_launches;
  if ((rc = launch_solve_pre(h, 0.0, s1))) { unavailable(cudaErrorUnknown); return rc; }
  k_lm_mark<<<1, 1, 0, s1>>>(S, 0);
  const int max_it = cfg->cg_max_iters;
  const double tol = cfg->cg_tol;
  if (gpcg) {
    k_g_setparams_lm<<<1, 1, 0, s1>>>(g, S, tol, max_it);
    if (ba) {
      k_g_init<<<CGV_BLOCKS, 256, 0, s1>>>(d, g);
      if (d.Gpm) { k_cam_wvec<<<h->cam_blocks, 256, 0, s1>>>(d, g.p, d.Wc); count_launch(h); }
      k_g_init2<<<1, 32, 0, s1>>>(d, g, CGV_BLOCKS);
    } else {
      k_gg_init<<<CGV_BLOCKS, 256, 0, s1>>>(h->gp, g);
      k_g_init2<<<1, 32, 0, s1>>>(h->gp, g, CGV_BLOCKS);
    }
    if ((e = cap_handle(s1, &hpcg))) return unavailable(e);
    k_g_cond_init<<<1, 1, 0, s1>>>(g, hpcg);
    count_launch(h, 5);
    if ((e = cap_cond(s1, hpcg, cudaGraphCondTypeWhile, &bpcg))) return unavailable(e);
    if (ba && !g.fused) set_l2_window(h, s2, d.yv, sizeof(double) * 4 * (size_t)d.bp.P);
    if ((e = cudaStreamBeginCaptureToGraph(s2, bpcg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)))
      return unavailable(e);
    if (ba) capture_ba_pcg_body(h, s2, hpcg);
    else capture_gp_pcg_body(h, s2, hpcg);
    if ((e = cudaStreamEndCapture(s2, &bpcg))) return unavailable(e);
  } else {
    double lam = 0.0;   // read from the device lambda by the kernel
    CGCtl* ctl = &h->misc->ctl;
    void* a[13];
    if (ba) a[0] = &d;
    else a[0] = &h->gp;
    a[1] = &h->fz; a[2] = &h->cm; a[3] = &lam; a[4] = (void*)&max_it; a[5] = (void*)&tol;
    a[6] = &h->x; a[7] = &h->r; a[8] = &h->z; a[9] = &h->p; a[10] = &h->q;
    a[11] = &h->part; a[12] = &ctl;
    if ((e = cudaLaunchCooperativeKernel(h->pcg_fn, dim3(h->pcg_grid), dim3(h->pcg_threads), a, h->pcg_smem, s1)))
      return unavailable(e);
    count_launch(h);
  }
  k_lm_mark<<<1, 1, 0, s1>>>(S, 1);
  if ((rc = launch_solve_post(h, s1))) { unavailable(cudaErrorUnknown); return rc; }
  k_axpy_theta<<<nblk(n, 256), 256, 0, s1>>>(h->theta, h->delta, h->cand, n);
  if ((rc = launch_post_step(h, h->cand, s1))) { unavailable(cudaErrorUnknown); return rc; }
  if ((rc = launch_cost(h, h->cand, s1))) { unavailable(cudaErrorUnknown); return rc; }
  k_lm_decide<CGCtl><<<1, 1, 0, s1>>>(S, &h->misc->status, &h->misc->ctl, scal + SC_COST, h->lrecs);
  k_lm_accept<<<std::min(nblk(n, 256), 4 * h->num_sms), 256, 0, s1>>>(S, h->cand, h->theta, n);
  h->lm_k_solve = h->prof.kernel_launches - k2 + 5;   // + marks, axpy, decide, accept
  if ((e = cudaStreamEndCapture(s1, &bsolve))) return unavailable(e);
  k_lm_tail<<<1, 1, 0, s0>>>(S, hw);
  h->lm_k_iter = 3;
  if ((e = cudaStreamEndCapture(s0, &body))) return unavailable(e);
  h->capturing = false;
  d.lamp = nullptr;
  h->gp.lamp = nullptr;
  h->prof.kernel_launches = k0;   // capture is not execution
  if ((e = cudaGraphInstantiate(&h->lm_exec, h->lm_graph, 0))) return unavailable(e);
  for (cudaStream_t x : {s0, s1, s2}) cudaStreamDestroy(x);
  h->lm_theta = h->theta;
  h->lm_cg_tol = tol;
  h->lm_cg_max = max_it;
  h->lm_state = 1;
  return SSFM_OK;
}

// lm_solve with the loop on the device: one graph launch, one read-back
static int lm_solve_graph(ssfm_handle* h, double* theta_io, const ssfm_lm_config* cfg, ssfm_iter_record* recs,
                          int32_t cap, int32_t* n_recs, int32_t* termination, cudaStream_t st) {
  if (h->lm_state == 1 && (h->lm_cg_tol != cfg->cg_tol || h->lm_cg_max != cfg->cg_max_iters ||
                           h->lrec_cap < cfg->max_iterations))
    destroy_lm_graph(h);
  if (h->lm_state == 0) {
    const auto tg = std::chrono::steady_clock::now();
    int rc = build_lm_graph(h, cfg);
    if (rc) return rc;
    if (getenv("SSFM_TIMING"))
      fprintf(stderr, "[ssfm] LM graph build %.1f ms (state %d)\n",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tg).count(), h->lm_state);
    if (h->lm_state != 1) return -1;   // unavailable: the caller runs the host loop
  }
  if (h->theta != h->lm_theta) std::swap(h->theta, h->cand);   // the captured buffers
  const long long n = h->total_params;
  LMState& H = *h->hlms;
  H.lambda0 = cfg->lambda0; H.lambda_up = cfg->lambda_up; H.lambda_down = cfg->lambda_down;
  H.lambda_min = cfg->lambda_min; H.lambda_max = cfg->lambda_max;
  H.rel_cost_tol = cfg->rel_cost_tol; H.grad_tol = cfg->grad_tol;
  H.max_it = cfg->max_iterations;
  H.cap = h->lrec_cap;
  CU(cudaMemcpyAsync(h->lms, h->hlms, sizeof(LMState), cudaMemcpyHostToDevice, st));
  CU(copy_async(h->theta, theta_io, n, st));
  h->prof.pcg_ms = h->prof.lin_ms = h->prof.all_ms = 0;
  h->prof.pcg_launches = h->prof.lin_launches = h->prof.all_launches = 0;
  h->prof.cg_iters = 0;
  h->prof.kernel_launches = 0;
  for (int k = 0; k < 5; ++k) h->prof.phase_ms[k] = 0;
  int rc = launch_cost(h, h->theta, st);
  if (rc) return rc;
  k_lm_init<<<1, 1, 0, st>>>(h->lms, (h->kind == 0 ? h->ba.scal : h->gp.scal) + SC_COST);
  count_launch(h);
  if (cfg->max_iterations >= 1) CU(cudaGraphLaunch(h->lm_exec, st));
  CU(cudaMemcpyAsync(h->hlms, h->lms, sizeof(LMState), cudaMemcpyDeviceToHost, st));
  CU(cudaMemcpyAsync(h->hlrecs, h->lrecs, sizeof(LMRecDev) * h->lrec_cap, cudaMemcpyDeviceToHost, st));
  CU(copy_async(theta_io, h->theta, n, st));
  CU(cudaStreamSynchronize(st));
  CU(cudaGetLastError());
  const LMState R = *h->hlms;
  const int nrec = std::min(R.nrec, h->lrec_cap);
  if (recs) {
    for (int k = 0; k < std::min(nrec, (int)cap); ++k) {
      const LMRecDev& D = h->hlrecs[k];
      ssfm_iter_record& O = recs[k];
      O.iteration = D.iteration;
      O.cost_before = D.cost_before;
      O.cost_after = D.cost_after;
      O.lam = D.lam;
      O.step_accepted = D.accepted;
      O.cg_iters = D.cg_iters;
      O.status = D.status;
      O.wall_time_ns = (int64_t)D.ns;   // device clock (no host round trip per iteration)
      O.device_ms = D.ns * 1e-6;
    }
  }
  for (int k = 0; k < nrec; ++k) {
    h->prof.pcg_ms += h->hlrecs[k].pcg_ns * 1e-6;
    h->prof.all_ms += h->hlrecs[k].ns * 1e-6;
  }
  h->prof.pcg_launches = nrec;
  h->prof.all_launches = nrec;
  h->prof.cg_iters = R.cg_total;
  count_launch(h, h->lm_k_iter * R.it + h->lm_k_lin * R.n_lin + h->lm_k_solve * R.n_solve +
                      (h->graph_state != -1 ? (long long)h->graph_body_kernels * R.cg_total : 0));
  if (R.n_lin > 0) h->linearized = true;
  if (n_recs) *n_recs = std::min(nrec, (int)cap);
  if (termination) *termination = R.term;
  if (R.result == SSFM_SOLVER_FAILURE) {
    Misc m = *h->hmisc;
    m.ctl.iters = R.fail_iters;
    m.ctl.rn = R.fail_rn;
    m.ctl.tol = R.fail_tol;
    set_err(SSFM_SOLVER_FAILURE, "linear solve failed at lambda_max: " + status_msg(R.fail_status, m));
    return SSFM_SOLVER_FAILURE;
  }
  return SSFM_OK;
}

extern "C" int ssfm_lm_solve(ssfm_handle* h, double* theta_io, const ssfm_lm_config* cfg,
                             ssfm_iter_record* recs, int32_t cap, int32_t* n_recs,
                             int32_t* termination, void* stream) {
  if (!h || !theta_io || !cfg) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  using clk = std::chrono::steady_clock;
  int rc;
  CU(zero_async(&h->misc->status, sizeof(int), st));
  if (lm_graph_wanted(h)) {
    rc = lm_solve_graph(h, theta_io, cfg, recs, cap, n_recs, termination, st);
    if (rc != -1) return rc;   // -1: no graph on this runtime, run the host loop
  }
  if (n_recs) *n_recs = 0;
  int term = SSFM_TERM_MAX_ITER;
  const long long n = h->total_params;
  CU(copy_async(h->theta, theta_io, n, st));
  if ((rc = launch_cost(h, h->theta, st))) return rc;
  if ((rc = read_misc(h, st))) return rc;
  double cost = h->hmisc->scal[SC_COST];
  double lam = cfg->lambda0;
  bool need_lin = true;
  int nrec = 0;
  h->prof.pcg_ms = h->prof.lin_ms = h->prof.all_ms = 0;
  h->prof.pcg_launches = h->prof.lin_launches = h->prof.all_launches = 0;
  h->prof.cg_iters = 0;
  h->prof.kernel_launches = 0;
  for (int k = 0; k < 5; ++k) h->prof.phase_ms[k] = 0;
  int result = SSFM_OK;
  for (int it = 1; it <= cfg->max_iterations; ++it) {
    auto t0 = clk::now();
    CU(cudaEventRecord(h->ev0, st));
    if (need_lin) {
      if ((rc = launch_linearize(h, h->theta, nullptr, nullptr, st))) return rc;
      // linearize-time gradient check needs the gradient max (lm.py:762)
      if ((rc = read_misc(h, st))) return rc;
      const double gmax = h->hmisc->scal[SC_GMAX];
      need_lin = false;
      if (gmax < cfg->grad_tol) { term = SSFM_TERM_CONVERGED_GRAD; break; }
    }
    if ((rc = launch_solve(h, lam, cfg, st))) return rc;
    // candidate = post_step(theta + delta); cost(candidate)
    k_axpy_theta<<<nblk(n, 256), 256, 0, st>>>(h->theta, h->delta, h->cand, n);
    count_launch(h);
    if ((rc = launch_post_step(h, h->cand, st))) return rc;
    if ((rc = launch_cost(h, h->cand, st))) return rc;
    if ((rc = sync_status(h, st))) return rc;
    CU(cudaEventRecord(h->ev1, st));
    if ((rc = read_misc(h, st))) return rc;
    const Misc m = *h->hmisc;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, h->ev0, h->ev1);
    if (h->prof.on) {
      float pms = 0.f;
      cudaEventElapsedTime(&pms, h->ev2, h->ev3);
      h->prof.pcg_ms += pms;
      h->prof.pcg_launches += 1;
      h->prof.cg_iters += m.ctl.iters;
      for (int k = 0; k < 5; ++k) h->prof.phase_ms[k] += m.ctl.phase_ns[k] * 1e-6;
    }
    if (h->graph_pending) {   // graph PCG: the WHILE body ran once per CG iteration (at least once)
      count_launch(h, h->graph_body_kernels * std::max(1, m.ctl.iters));
      h->graph_pending = false;
    }
    const int code = status_to_code(m.status);
    if (code == SSFM_COMM_ERROR) {   // a peer did not answer: the exchanged values are not valid
      CU(copy_async(theta_io, h->theta, n, st));
      CU(cudaStreamSynchronize(st));
      if (n_recs) *n_recs = std::min(nrec, (int)cap);
      return set_err(SSFM_COMM_ERROR, status_msg(m.status, m));
    }
    const bool pcg_done = !(m.status & (ST_SINGULAR_POINT | ST_PIN_POINT | ST_SINGULAR_PRECOND |
                                        ST_PIN_RETAINED | ST_PIN_SCALE | ST_CG_MAXITER | ST_CG_BREAKDOWN));
    double cost_new = NAN;
    bool failed = code != SSFM_OK;
    if (failed) {
      if (lam >= cfg->lambda_max) {
        term = SSFM_TERM_SOLVER_FAILURE;
        set_err(SSFM_SOLVER_FAILURE, "linear solve failed at lambda_max: " + status_msg(m.status, m));
        result = SSFM_SOLVER_FAILURE;
        break;
      }
    } else {
      cost_new = m.scal[SC_COST];
    }
    const bool accepted = !failed && std::isfinite(cost_new) && cost_new < cost;
    if (recs && nrec < cap) {
      ssfm_iter_record& R = recs[nrec];
      R.iteration = it;
      R.cost_before = cost;
      R.cost_after = cost_new;
      R.lam = lam;
      R.step_accepted = accepted;
      R.cg_iters = pcg_done ? m.ctl.iters : 0;
      R.status = code;
      R.wall_time_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(clk::now() - t0).count();
      R.device_ms = ms;
    }
    ++nrec;
    h->prof.all_ms += ms;
    h->prof.all_launches += 1;
    if (accepted) {
      const double rel = (cost - cost_new) / std::max(cost, 1e-300);
      std::swap(h->theta, h->cand);
      cost = cost_new;
      lam = std::max(lam / cfg->lambda_down, cfg->lambda_min);
      need_lin = true;
      if (rel < cfg->rel_cost_tol) { term = SSFM_TERM_CONVERGED_COST; break; }
    } else {
      lam = std::min(lam * cfg->lambda_up, cfg->lambda_max);
    }
  }
  CU(copy_async(theta_io, h->theta, n, st));
  CU(cudaStreamSynchronize(st));
  if (n_recs) *n_recs = std::min(nrec, (int)cap);
  if (termination) *termination = term;
  return result;
}

extern "C" int32_t ssfm_lm_mode(const ssfm_handle* h) { return h ? h->lm_state : 0; }

extern "C" int ssfm_profile_enable(ssfm_handle* h, int32_t on) {
  if (!h) return SSFM_INVALID_ARGUMENT;
  h->prof.on = on != 0;
  return SSFM_OK;
}

extern "C" int ssfm_profile_get(const ssfm_handle* h, int32_t kind, double* ms, int64_t* launches,
                                double* bytes) {
  if (!h) return SSFM_INVALID_ARGUMENT;
  const Profile& p = h->prof;
  if (kind == 0) {
    if (ms) *ms = p.pcg_ms;
    if (launches) *launches = p.pcg_launches;
    if (bytes) *bytes = (double)p.cg_iters;
  } else if (kind == 1) {
    if (ms) *ms = p.lin_ms;
    if (launches) *launches = p.lin_launches;
    if (bytes) *bytes = 0;
  } else if (kind >= 3 && kind <= 7) {
    if (ms) *ms = p.phase_ms[kind - 3];
    if (launches) *launches = p.pcg_launches;
    if (bytes) *bytes = 0;
  } else {
    if (ms) *ms = p.all_ms;
    if (launches) *launches = p.kernel_launches;
    if (bytes) *bytes = 0;
  }
  return SSFM_OK;
}

extern "C" int ssfm_comm_init(ssfm_handle* h, int32_t rank, int32_t nranks, void* ipc_handle_out,
                              void** region_out) {
  if (!h) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  if (nranks < 1 || nranks > SSFM_MAX_RANKS || rank < 0 || rank >= nranks)
    return set_err(SSFM_INVALID_ARGUMENT, "bad rank / nranks");
  if (h->region) return set_err(SSFM_INVALID_ARGUMENT, "exchange region already initialised");
  const int C = h->topo.C;
  const int per_cam = h->kind == 0 ? std::max(CAM_V, 8) : std::max(GPE_V, 4);
  const long long cap = (long long)per_cam * C + 64;
  const size_t bytes = 256 + sizeof(double) * 2 * (size_t)cap;
  CU(cudaMalloc(&h->region, bytes));
  CU(cudaMemset(h->region, 0, bytes));
  DALLOC(h->cm.epoch, 1);
  CU(cudaMemset(h->cm.epoch, 0, sizeof(unsigned long long)));
  DALLOC(h->camsum, (long long)per_cam * C);
  DALLOC(h->ar_tmp, 16);
  CU(cudaDeviceSynchronize());
  CommDev& cm = h->cm;
  cm.rank = rank;
  cm.cap = cap;
  cm.flag[rank] = static_cast<unsigned long long*>(h->region);
  cm.buf[rank] = reinterpret_cast<double*>(static_cast<char*>(h->region) + 256);
  cm.status = &h->misc->status;
  if (const char* e = getenv("SSFM_COMM_TIMEOUT_S")) {
    const double sec = atof(e);
    if (sec > 0) cm.timeout_ns = (unsigned long long)(sec * 1e9);
  }
  cm.nranks = 1;   // becomes nranks on connect
  h->comm_nranks = nranks;
  if (ipc_handle_out) {
    cudaIpcMemHandle_t ih;
    CU(cudaIpcGetMemHandle(&ih, h->region));
    memcpy(ipc_handle_out, &ih, sizeof(ih));
  }
  if (region_out) *region_out = h->region;
  return SSFM_OK;
}

extern "C" int ssfm_comm_connect(ssfm_handle* h, const void* ipc_handles, void* const* regions) {
  if (!h || !h->region) return set_err(SSFM_INVALID_ARGUMENT, "ssfm_comm_connect before ssfm_comm_init");
  if (!ipc_handles && !regions) return set_err(SSFM_INVALID_ARGUMENT, "need IPC handles or region pointers");
  CommDev& cm = h->cm;
  const int R = h->comm_nranks;
  for (int r = 0; r < R; ++r) {
    if (r == cm.rank) continue;
    void* ptr = nullptr;
    if (regions && regions[r]) {
      ptr = regions[r];
    } else if (ipc_handles) {
      cudaIpcMemHandle_t ih;
      memcpy(&ih, static_cast<const char*>(ipc_handles) + sizeof(ih) * r, sizeof(ih));
      cudaError_t e = cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess)
        return set_err(SSFM_COMM_ERROR, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
      h->ipc_opened.push_back(ptr);
    } else {
      return set_err(SSFM_INVALID_ARGUMENT, "missing peer region");
    }
    cm.flag[r] = static_cast<unsigned long long*>(ptr);
    cm.buf[r] = reinterpret_cast<double*>(static_cast<char*>(ptr) + 256);
  }
  cm.nranks = R;
  // build the graph PCG now, from the connecting thread: building it inside
  // the first solve would allocate device memory while a peer shard's kernel
  // may already wait in an exchange. With several shards on one device, a
  // device allocation (like a NULL-stream command) serialises the streams
  // around it, so the peer would wait for this shard's kernels forever.
  if (h->kind == 0 && h->graph_state == 1 && !h->graph_sharded) {
    cudaGraphExecDestroy(h->pcg_exec);
    cudaGraphDestroy(h->pcg_graph);
    h->pcg_exec = nullptr;
    h->pcg_graph = nullptr;
    h->graph_state = 0;
  }
  if (h->kind == 0 && h->graph_state == 0) {
    int rc = build_pcg_graph(h);
    if (rc) return rc;
    h->graph_sharded = true;
  }
  return SSFM_OK;
}

extern "C" int32_t ssfm_handle_device(const ssfm_handle* h) { return h ? h->device : -1; }

// Peer access from `device` to `peer` (several devices driven by one process,
// dist.connect_local): the exchange regions of the other devices' handles are
// then read and written directly over NVLink.
extern "C" int ssfm_enable_peer_access(int32_t device, int32_t peer) {
  if (device == peer) return SSFM_OK;
  int can = 0;
  CU(cudaDeviceCanAccessPeer(&can, device, peer));
  if (!can) return set_err(SSFM_COMM_ERROR, "device " + std::to_string(device) + " cannot access device " +
                                                std::to_string(peer) + " (no peer access)");
  int cur = 0;
  CU(cudaGetDevice(&cur));
  CU(cudaSetDevice(device));
  cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) { cudaGetLastError(); e = cudaSuccess; }
  cudaSetDevice(cur);
  if (e != cudaSuccess) return set_err(SSFM_COMM_ERROR, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
  return SSFM_OK;
}

extern "C" int ssfm_check_jacobian(ssfm_handle* h, int64_t* mismatches, void* stream) {
  if (!h || !mismatches) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  if (h->kind != 0) return set_err(SSFM_INVALID_ARGUMENT, "BA handles only");
  if (!h->linearized) return set_err(SSFM_INVALID_ARGUMENT, "ssfm_check_jacobian before ssfm_linearize");
  if (!h->ba.Jcm)
    return set_err(SSFM_INVALID_ARGUMENT, "no camera-major Jacobian copy: this handle's camera pass reads the "
                                          "factored record (SSFM_FACTORED=0 keeps the copy)");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* dm = nullptr;
  CU(cudaMalloc(&dm, sizeof(unsigned long long)));
  CU(cudaMemsetAsync(dm, 0, sizeof(unsigned long long), st));
  k_check_jcopies<<<nblk(h->topo.N, 256), 256, 0, st>>>(h->ba, dm);
  unsigned long long hm = 0;
  cudaMemcpyAsync(&hm, dm, sizeof(hm), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(dm);
  CU(cudaGetLastError());
  *mismatches = (int64_t)hm;
  return SSFM_OK;
}

// GP passes as standalone kernels (per-pass timing / ncu, ssfm_bench_operator)
__global__ void __launch_bounds__(PCG_THREADS, 4) k_gop_point(GPDev d, const double* v, double* y) {
  __shared__ double smp[PCG_THREADS / 32][SSFM_BATCH][3];
  gp_point_pass(d, v, y, smp);
}
__global__ void __launch_bounds__(PCG_THREADS, 4) k_gop_camera(GPDev d, const double* y, double* tile4) {
  __shared__ double smred[(PCG_THREADS / 32) * 8];
  gp_camera_pass(d, y, tile4, smred);
}

static int bench_operator_gp(ssfm_handle* h, int32_t which, int32_t reps, double* ms_out, cudaStream_t st) {
  GPDev& d = h->gp;
  int occ_p = 0, occ_c = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_p, (const void*)k_gop_point, PCG_THREADS, 0));
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_c, (const void*)k_gop_camera, PCG_THREADS, 0));
  auto run = [&]() {
    if (which != 1) k_gop_point<<<std::max(1, occ_p) * h->num_sms, PCG_THREADS, 0, st>>>(d, h->p, d.yv);
    if (which != 0 && d.topo.nt) k_gop_camera<<<std::max(1, occ_c) * h->num_sms, PCG_THREADS, 0, st>>>(d, d.yv, d.tilebuf);
  };
  for (int w = 0; w < 2; ++w) run();
  CU(cudaEventRecord(h->ev0, st));
  for (int k = 0; k < reps; ++k) run();
  CU(cudaEventRecord(h->ev1, st));
  CU(cudaEventSynchronize(h->ev1));
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  *ms_out = ms / reps;
  return SSFM_OK;
}

extern "C" int ssfm_bench_operator(ssfm_handle* h, int32_t which, int32_t reps, double* ms_out, void* stream) {
  if (!h || !ms_out || reps < 1) return set_err(SSFM_INVALID_ARGUMENT, "bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  if (h->kind == 1) return bench_operator_gp(h, which, reps, ms_out, st);
  BADev& d = h->ba;
  const bool fac = d.Fcm != nullptr;
  const void* fn = which != 1 ? (const void*)k_op_point
                              : (fac ? (const void*)k_op_camera<true> : (const void*)k_op_camera<false>);
  int occ = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, which != 1 ? PTP_THREADS : PCG_THREADS, 0));
  const int grid = std::max(1, occ) * h->num_sms;
  int occ2 = 0;
  const void* fn2 = fac ? (const void*)k_op_camera<true> : (const void*)k_op_camera<false>;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, fn2, PCG_THREADS, 0));
  const int grid2 = std::max(1, occ2) * h->num_sms;
  auto run = [&]() {
    if (which == 0) {
      k_op_point<<<grid, PTP_THREADS, 0, st>>>(d, h->p, d.yv);
    } else if (which == 2) {   // the operator's two passes back to back (as in the PCG)
      k_op_point<<<grid, PTP_THREADS, 0, st>>>(d, h->p, d.yv);
      if (fac) k_op_camera<true><<<grid2, PCG_THREADS, 0, st>>>(d, d.yv, d.tilebuf);
      else k_op_camera<false><<<grid2, PCG_THREADS, 0, st>>>(d, d.yv, d.tilebuf);
    } else {
      if (fac) k_op_camera<true><<<grid, PCG_THREADS, 0, st>>>(d, d.yv, d.tilebuf);
      else k_op_camera<false><<<grid, PCG_THREADS, 0, st>>>(d, d.yv, d.tilebuf);
    }
  };
  if (d.Gpm) k_cam_wvec<<<h->cam_blocks, 256, 0, st>>>(d, h->p, d.Wc);   // omega form: W of p
  const bool win = set_l2_window(h, st, d.yv, sizeof(double) * 4 * (size_t)d.bp.P);
  for (int w = 0; w < 2; ++w) run();   // warm-up
  CU(cudaEventRecord(h->ev0, st));
  for (int k = 0; k < reps; ++k) run();
  CU(cudaEventRecord(h->ev1, st));
  CU(cudaEventSynchronize(h->ev1));
  if (win) clear_l2_window(st);
  float ms = 0.f;
  CU(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  *ms_out = ms / reps;
  return SSFM_OK;
}

__global__ void k_sum_pairs(const double* __restrict__ part, int n, double* out) {
  __shared__ double sm[64];
  double v[2] = {0.0, 0.0};
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int a = threadIdx.x * per, b = min(n, a + per);
  for (int k = a; k < b; ++k) { v[0] += part[2ll * k]; v[1] += part[2ll * k + 1]; }
  block_reduce<2>(v, sm);
  if (threadIdx.x == 0) { out[0] = v[0]; out[1] = v[1]; }
}

extern "C" int ssfm_reproj_stats(ssfm_handle* h, const double* theta, double* sum_sq, int64_t* count,
                                 void* stream) {
  if (!h || !theta) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  if (h->kind != 0) return set_err(SSFM_INVALID_ARGUMENT, "BA handles only");
  cudaStream_t st = (cudaStream_t)stream;
  BADev& d = h->ba;
  const int nb = nblk(h->topo.N, 256);
  double* part = nullptr;
  CU(cudaMalloc(&part, sizeof(double) * (2ll * nb + 2)));
  ba_k_prep<<<h->cam_blocks, 256, 0, st>>>(d, theta);
  ba_k_reproj<<<nb, 256, 0, st>>>(d, theta, part);
  k_sum_pairs<<<1, 1024, 0, st>>>(part, nb, part + 2ll * nb);
  double hv[2] = {0.0, 0.0};
  cudaMemcpyAsync(hv, part + 2ll * nb, sizeof(hv), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(part);
  CU(cudaGetLastError());
  if (sum_sq) *sum_sq = hv[0];
  if (count) *count = (int64_t)hv[1];
  return SSFM_OK;
}

// ---------------------------------------------------------------------------
// generic block algebra (sparse_block.jtj / jtr / apply_damping)
// ---------------------------------------------------------------------------
extern "C" int ssfm_block_jtj(const double* entry_data, const int64_t* entry_off, const int32_t* entry_h,
                              const int32_t* entry_w, const int64_t* contrib_a, const int64_t* contrib_b,
                              const int64_t* seg_start, const int64_t* key_out_off, int64_t nkeys,
                              double* out_data, void* stream) {
  if (nkeys < 0) return set_err(SSFM_INVALID_ARGUMENT, "negative key count");
  if (nkeys == 0) return SSFM_OK;
  if (!entry_data || !entry_off || !entry_h || !entry_w || !contrib_a || !contrib_b || !seg_start ||
      !key_out_off || !out_data)
    return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  k_block_jtj<<<nblk(nkeys, 128), 128, 0, (cudaStream_t)stream>>>(
      entry_data, (const long long*)entry_off, entry_h, entry_w, (const long long*)contrib_a,
      (const long long*)contrib_b, (const long long*)seg_start, (const long long*)key_out_off, nkeys, out_data);
  CU(cudaGetLastError());
  return SSFM_OK;
}

extern "C" int ssfm_block_jtr(const double* entry_data, const int64_t* entry_off, const int32_t* entry_h,
                              const int32_t* entry_w, const int32_t* by_entry, const int64_t* seg_start,
                              const int64_t* seg_out, const int64_t* res_row, int64_t nsegs,
                              const double* residuals, double* out, void* stream) {
  if (nsegs < 0) return set_err(SSFM_INVALID_ARGUMENT, "negative segment count");
  if (nsegs == 0) return SSFM_OK;
  if (!entry_data || !entry_off || !entry_h || !entry_w || !by_entry || !seg_start || !seg_out || !res_row ||
      !residuals || !out)
    return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  k_block_jtr<<<nblk(nsegs, 128), 128, 0, (cudaStream_t)stream>>>(
      entry_data, (const long long*)entry_off, entry_h, entry_w, by_entry, (const long long*)seg_start,
      (const long long*)seg_out, (const long long*)res_row, nsegs, residuals, out);
  CU(cudaGetLastError());
  return SSFM_OK;
}

extern "C" int ssfm_block_scale_diag(double* data, const int64_t* diag_idx, int64_t n, double factor,
                                     void* stream) {
  if (n < 0) return set_err(SSFM_INVALID_ARGUMENT, "negative count");
  if (n == 0) return SSFM_OK;
  if (!data || !diag_idx) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  k_block_scale_diag<<<nblk(n, 256), 256, 0, (cudaStream_t)stream>>>(data, (const long long*)diag_idx, n, factor);
  CU(cudaGetLastError());
  return SSFM_OK;
}

// ---------------------------------------------------------------------------
// Schur PCG on an explicit block normal system (schur_explicit.cuh)
// ---------------------------------------------------------------------------
extern "C" int ssfm_trim_cache(int32_t device, int64_t* freed_bytes) {
  const size_t f = block_cache_trim(device);
  if (freed_bytes) *freed_bytes = (int64_t)f;
  return SSFM_OK;
}

extern "C" int64_t ssfm_cache_bytes(void) {
  BlockCache& bc = block_cache();
  std::lock_guard<std::mutex> lk(bc.mu);
  return (int64_t)bc.bytes;
}

extern "C" int ssfm_schur_solve(const ssfm_schur_plan* plan, const double* data, const double* gradient,
                                const ssfm_lm_config* cfg, double* delta, int32_t* cg_iters_host, void* stream) {
  if (!plan || !data || !gradient || !cfg || !delta) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  const XsPlan& pl = *plan;
  if (pl.n_params <= 0 || pl.n_ret < 0 || pl.n_pt < 0 || pl.n_u < 0 || pl.n_sc < 0)
    return set_err(SSFM_INVALID_ARGUMENT, "bad plan sizes");
  cudaStream_t st = (cudaStream_t)stream;
  const long long n = pl.n_ret;
  long long nu_sc = 0, npre = 0;
  if (pl.n_u) CU(cudaMemcpyAsync(&nu_sc, pl.u_off + pl.n_u, sizeof(long long), cudaMemcpyDeviceToHost, st));
  if (pl.n_rblk) CU(cudaMemcpyAsync(&npre, pl.pre_off + pl.n_rblk, sizeof(long long), cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  // one stream-ordered scratch block: S | U | dpt | M | y | g | bred x r z p q | prec | ctl + status
  const long long nd = n * n + nu_sc + 9 * pl.n_pt * 2 + 3 * pl.n_pt + pl.n_params + 6 * n + npre + 8;
  double* base = nullptr;
  CU(cudaMallocAsync((void**)&base, sizeof(double) * nd, st));
  XsWork w{};
  double* c = base;
  w.S = c; c += n * n;
  w.U = c; c += nu_sc;
  w.dpt = c; c += 9 * pl.n_pt;
  w.M = c; c += 9 * pl.n_pt;
  w.y = c; c += 3 * pl.n_pt;
  w.g = c; c += pl.n_params;
  w.bred = c; c += n;
  w.x = c; c += n;
  w.r = c; c += n;
  w.z = c; c += n;
  w.p = c; c += n;
  w.q = c; c += n;
  w.prec = c; c += npre;
  w.ctl = (XsWork::Ctl*)c;
  w.status = (int*)(c + 6);
  int rc = SSFM_OK;
  auto finish = [&](int code) {
    cudaFreeAsync(base, st);
    return code;
  };
  if (cudaMemsetAsync(w.S, 0, sizeof(double) * n * n, st) || cudaMemsetAsync(c, 0, sizeof(double) * 8, st))
    return finish(set_err(SSFM_CUDA_ERROR, "memset"));
  const int T = 256;
  const long long big = std::max(std::max<long long>(pl.n_direct, nu_sc), std::max<long long>(9 * pl.n_pt, std::max<long long>(pl.n_params, 1)));
  k_xs_init<<<(int)std::min<long long>(nblk(big, T), 148 * 16), T, 0, st>>>(pl, data, gradient, w);
  if (pl.n_sc) {
    k_xs_sc_check<<<nblk(pl.n_sc, T), T, 0, st>>>(pl, data, gradient, w);
    if (pl.n_rblk) k_xs_sc_cam<<<nblk(pl.n_rblk, T), T, 0, st>>>(pl, data, gradient, w);
    if (pl.n_pt) k_xs_sc_pt<<<nblk(pl.n_pt, T), T, 0, st>>>(pl, data, gradient, w);
    if (pl.n_u) k_xs_sc_u<<<nblk(pl.n_u, T), T, 0, st>>>(pl, data, w);
  }
  if (pl.n_pt) k_xs_ptinv<<<nblk(pl.n_pt, T), T, 0, st>>>(pl, w);
  if (pl.n_rblk) k_xs_bred<<<nblk(pl.n_rblk, T), T, 0, st>>>(pl, w);
  if (pl.n_slots) k_xs_fill<<<nblk(32 * pl.n_slots, T), T, 0, st>>>(pl, w);
  if (n) k_xs_pin<<<nblk(n, T), T, 0, st>>>(pl, w);
  if (pl.n_rblk) k_xs_prec<<<nblk(pl.n_rblk, 64), 64, 0, st>>>(pl, w);
  int status = 0;
  if (cudaGetLastError() != cudaSuccess) return finish(set_err(SSFM_CUDA_ERROR, "schur setup launch failed"));
  if (cudaMemcpyAsync(&status, w.status, sizeof(int), cudaMemcpyDeviceToHost, st) || cudaStreamSynchronize(st))
    return finish(set_err(SSFM_CUDA_ERROR, "schur setup failed"));
  // the reference raises in this order (lm.py:569-575, 503-512, 631-633, 520-525)
  if (status & ST_PIN_SCALE) return finish(set_err(SSFM_SINGULAR_BLOCK, "masked scale with non-zero coupling"));
  if (status & ST_PIN_POINT)
    return finish(set_err(SSFM_SINGULAR_BLOCK, "masked point direction with non-zero gradient"));
  if (status & ST_SINGULAR_POINT)
    return finish(set_err(SSFM_SINGULAR_BLOCK, "eliminable block singular after damping (det <= 0)"));
  if (status & ST_PIN_RETAINED)
    return finish(set_err(SSFM_SINGULAR_BLOCK, "masked retained direction with non-zero gradient"));
  if (status & ST_SINGULAR_PRECOND)
    return finish(set_err(SSFM_SINGULAR_BLOCK, "singular preconditioner block"));
  // PCG: the iterations are enqueued in chunks; a finished solve turns the
  // remaining kernels of the chunk into no-ops, so the count is exact
  k_xs_cg_start<<<1, 1024, 0, st>>>(pl, w, gradient, cfg->cg_tol, cfg->cg_max_iters);
  XsWork::Ctl hc{};
  const int chunk = 16;
  const int mv_blocks = nblk(32 * std::max<long long>(n, 1), T);
  for (;;) {
    if (cudaMemcpyAsync(&hc, w.ctl, sizeof(hc), cudaMemcpyDeviceToHost, st) || cudaStreamSynchronize(st))
      return finish(set_err(SSFM_CUDA_ERROR, "schur PCG failed"));
    if (hc.done) break;
    for (int k = 0; k < chunk; ++k) {
      k_xs_matvec<<<mv_blocks, T, 0, st>>>(pl, w);
      k_xs_cg_step<<<1, 1024, 0, st>>>(pl, w);
    }
    if (cudaGetLastError() != cudaSuccess) return finish(set_err(SSFM_CUDA_ERROR, "schur PCG launch failed"));
  }
  if (cg_iters_host) *cg_iters_host = hc.iters;
  char msg[160];
  if (hc.done == 2) {
    snprintf(msg, sizeof msg, "CG did not reach tolerance in %d iterations (|r| %.3e, tol %.3e)", hc.cg_max, hc.rn,
             hc.tol);
    return finish(set_err(SSFM_CG_STALL, msg));
  }
  if (hc.done == 3) return finish(set_err(SSFM_CG_STALL, "CG broke down (p.q <= 0 or non-finite)"));
  k_xs_back_zero<<<(int)std::min<long long>(nblk(pl.n_params, T), 148 * 8), T, 0, st>>>(pl, delta);
  if (n) k_xs_back_x<<<nblk(n, T), T, 0, st>>>(pl, w, delta);
  if (pl.n_pt) k_xs_back_pt<<<nblk(pl.n_pt, T), T, 0, st>>>(pl, w, delta);
  if (pl.n_sc) k_xs_back_sc<<<nblk(pl.n_sc, T), T, 0, st>>>(pl, data, gradient, delta);
  if (cudaGetLastError() != cudaSuccess) return finish(set_err(SSFM_CUDA_ERROR, "schur back-substitution failed"));
  rc = finish(SSFM_OK);
  return rc;
}

extern "C" int ssfm_dense_scatter(const double* data, const int64_t* dst, const int64_t* src, int64_t m,
                                  double* A, void* stream) {
  if (m < 0) return set_err(SSFM_INVALID_ARGUMENT, "negative count");
  if (m == 0) return SSFM_OK;
  if (!data || !dst || !src || !A) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  k_dense_scatter<<<nblk(m, 256), 256, 0, (cudaStream_t)stream>>>(data, (const long long*)dst,
                                                                 (const long long*)src, m, A);
  CU(cudaGetLastError());
  return SSFM_OK;
}

extern "C" int ssfm_dense_solve(double* A, const double* b, double* x, int64_t n, void* stream) {
  if (!A || !b || !x || n <= 0) return set_err(SSFM_INVALID_ARGUMENT, "bad argument");
  if (n > (1ll << 31) - 1) return set_err(SSFM_INVALID_ARGUMENT, "dense system too large");
  CuSolverApi& api = cusolver_api();
  if (!api.ok) return set_err(SSFM_CUDA_ERROR, "cuSOLVER (libcusolver.so.11) unavailable");
  cudaStream_t st = (cudaStream_t)stream;
  double *s = nullptr, *rhs = nullptr, *work = nullptr;
  int *flag = nullptr, *devinfo = nullptr;
  CU(cudaMalloc(&s, sizeof(double) * n));
  CU(cudaMalloc(&rhs, sizeof(double) * n));
  CU(cudaMalloc(&flag, sizeof(int) * 2));
  devinfo = flag + 1;
  CU(cudaMemsetAsync(flag, 0, sizeof(int) * 2, st));
  k_dense_prep<<<nblk(n, 256), 256, 0, st>>>(A, b, n, s, rhs, flag);
  k_dense_scale<<<nblk(n * n, 256), 256, 0, st>>>(A, s, n);
  cusolverDnHandle_t hs = nullptr;
  int rc = SSFM_OK;
  int lwork = 0, hflag[2] = {0, 0};
  if (api.create(&hs) != CUSOLVER_STATUS_SUCCESS) rc = set_err(SSFM_CUDA_ERROR, "cusolverDnCreate failed");
  if (!rc) api.set_stream(hs, st);
  if (!rc && api.potrf_bs(hs, CUBLAS_FILL_MODE_LOWER, (int)n, A, (int)n, &lwork) != CUSOLVER_STATUS_SUCCESS)
    rc = set_err(SSFM_CUDA_ERROR, "potrf_bufferSize failed");
  if (!rc && cudaMalloc(&work, sizeof(double) * std::max(lwork, 1))) rc = set_err(SSFM_CUDA_ERROR, "cudaMalloc");
  if (!rc && api.potrf(hs, CUBLAS_FILL_MODE_LOWER, (int)n, A, (int)n, work, lwork, devinfo) != CUSOLVER_STATUS_SUCCESS)
    rc = set_err(SSFM_CUDA_ERROR, "potrf failed");
  if (!rc) {
    cudaMemcpyAsync(hflag, flag, sizeof(hflag), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    if (hflag[0] & 1) rc = set_err(SSFM_SINGULAR_BLOCK, "zero diagonal with non-zero gradient");
    else if (hflag[0] & 2) rc = set_err(SSFM_SINGULAR_BLOCK, "negative diagonal in damped system");
    else if (hflag[1] != 0) rc = set_err(SSFM_SINGULAR_BLOCK, "dense factorization failed (potrf info " +
                                                            std::to_string(hflag[1]) + ")");
  }
  if (!rc && api.potrs(hs, CUBLAS_FILL_MODE_LOWER, (int)n, 1, A, (int)n, rhs, (int)n, devinfo) != CUSOLVER_STATUS_SUCCESS)
    rc = set_err(SSFM_CUDA_ERROR, "potrs failed");
  if (!rc) k_dense_unscale<<<nblk(n, 256), 256, 0, st>>>(s, rhs, n, x);
  cudaStreamSynchronize(st);
  if (hs) api.destroy(hs);
  cudaFree(s); cudaFree(rhs); cudaFree(flag);
  if (work) cudaFree(work);
  if (!rc && cudaGetLastError() != cudaSuccess) rc = set_err(SSFM_CUDA_ERROR, "dense solve kernel failed");
  return rc;
}

extern "C" int ssfm_operator_info(const ssfm_handle* h, int32_t* slot_groups, int32_t* grid,
                                  int32_t* threads, int64_t* smem_bytes) {
  if (!h) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  if (slot_groups) *slot_groups = h->fz.G;
  if (grid) *grid = h->pcg_grid;
  if (threads) *threads = h->pcg_threads;
  if (smem_bytes) *smem_bytes = (int64_t)h->pcg_smem;
  return SSFM_OK;
}

extern "C" int ssfm_export_pattern(ssfm_handle* h, int32_t* obs_pt_order, int32_t* obs_cam_order,
                                   int32_t* off_keys, int64_t off_cap, int64_t* n_off, int32_t* slots,
                                   int64_t slot_cap, int64_t* n_slots, void* stream) {
  if (!h) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const long long N = h->topo.N;
  if (obs_pt_order) CU(cudaMemcpyAsync(obs_pt_order, h->topo.pm_obs, sizeof(int) * N, cudaMemcpyDeviceToDevice, st));
  if (obs_cam_order) CU(cudaMemcpyAsync(obs_cam_order, h->topo.cm_obs, sizeof(int) * N, cudaMemcpyDeviceToDevice, st));
  int rc = export_keys(h, off_keys, off_cap, n_off, slots, slot_cap, n_slots, st);
  if (rc) return rc;
  CU(cudaStreamSynchronize(st));
  return SSFM_OK;
}

// ---------------------------------------------------------------------------
// accuracy metrics (synth_metrics.py:210-309), device-resident scenes
// ---------------------------------------------------------------------------
extern "C" int ssfm_rotation_auc(const double* q_est, const double* q_true, int32_t C, const double* taus,
                                 int32_t ntau, double* auc, void* stream) {
  if (!q_est || !q_true || !taus || !auc) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  if (C < 2) return set_err(SSFM_INVALID_ARGUMENT, "need >= 2 cameras");
  if (ntau < 1 || ntau > MET_MAX_TAU) return set_err(SSFM_INVALID_ARGUMENT, "1..16 thresholds");
  AucArgs a{};
  a.ntau = ntau;
  for (int k = 0; k < ntau; ++k) {
    if (!(taus[k] > 0.0)) return set_err(SSFM_INVALID_ARGUMENT, "thresholds must be positive");
    a.inv_tau[k] = 1.0 / taus[k];
  }
  cudaStream_t st = (cudaStream_t)stream;
  double* buf = nullptr;
  const long long rows = C - 1;
  CU(cudaMalloc(&buf, sizeof(double) * (8ll * C + MET_MAX_TAU * rows + MET_MAX_TAU)));
  double *ne = buf, *nt = buf + 4ll * C, *part = buf + 8ll * C, *res = part + MET_MAX_TAU * rows;
  k_met_qnorm<<<nblk(2ll * C, 256), 256, 0, st>>>(q_est, q_true, C, ne, nt);
  k_met_auc_rows<<<(int)rows, MET_THREADS, 0, st>>>(ne, nt, C, a, part);
  k_met_auc_final<<<1, 32, 0, st>>>(part, (int)rows, ntau, res);
  double hv[MET_MAX_TAU];
  cudaMemcpyAsync(hv, res, sizeof(double) * ntau, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(buf);
  CU(cudaGetLastError());
  const double npairs = 0.5 * (double)C * (double)(C - 1);
  for (int k = 0; k < ntau; ++k) auc[k] = hv[k] / npairs * 100.0;
  return SSFM_OK;
}

extern "C" int ssfm_center_moments(const double* x, const double* y, int32_t n, double* out, void* stream) {
  if (!x || !y || !out) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  if (n < 1) return set_err(SSFM_INVALID_ARGUMENT, "need >= 1 camera");
  cudaStream_t st = (cudaStream_t)stream;
  double* d = nullptr;
  CU(cudaMalloc(&d, sizeof(double) * 17));
  k_met_moments<<<1, 1024, 0, st>>>(x, y, n, d);
  cudaMemcpyAsync(out, d, sizeof(double) * 17, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(d);
  CU(cudaGetLastError());
  return SSFM_OK;
}

extern "C" int ssfm_apply_sim3(const double* rot, const double* trans, double scale, const double* rq_conj,
                               double* quats, double* centers, int32_t C, double* points, int64_t P,
                               void* stream) {
  if (!rot || !trans || !rq_conj) return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  if ((C > 0 && (!quats || !centers)) || (P > 0 && !points) || C < 0 || P < 0)
    return set_err(SSFM_INVALID_ARGUMENT, "bad scene arrays");
  Sim3Args a{};
  for (int k = 0; k < 9; ++k) a.R[k] = rot[k];
  for (int k = 0; k < 3; ++k) a.t[k] = trans[k];
  for (int k = 0; k < 4; ++k) a.rqc[k] = rq_conj[k];
  a.s = scale;
  cudaStream_t st = (cudaStream_t)stream;
  if (C > 0) k_met_apply_cameras<<<nblk(C, 256), 256, 0, st>>>(a, quats, centers, C);
  if (P > 0) k_met_apply_points<<<nblk(P, 256), 256, 0, st>>>(a, points, P);
  CU(cudaGetLastError());
  return SSFM_OK;
}

extern "C" int ssfm_make_rays(int64_t n, const int64_t* cam_idx, const double* pixels, const double* pps,
                              const double* focals, const double* quats, const double* depths, double* rays,
                              double* ray_depths, void* stream) {
  if (n < 0) return set_err(SSFM_INVALID_ARGUMENT, "negative observation count");
  if (n == 0) return SSFM_OK;
  if (!cam_idx || !pixels || !pps || !focals || !quats || !rays || (depths && !ray_depths))
    return set_err(SSFM_INVALID_ARGUMENT, "null argument");
  k_make_rays<<<nblk(n, 256), 256, 0, (cudaStream_t)stream>>>(n, (const long long*)cam_idx, pixels, pps, focals,
                                                              quats, depths, rays, ray_depths);
  CU(cudaGetLastError());
  return SSFM_OK;
}

// ba.prune (ba.py:223-261) on the device (csrc/prune.cuh). Inputs and outputs
// are device arrays; camera_map [C], point_map [P] (int32, -1 = removed),
// obs_mask [N] (uint8). Returns SSFM_EMPTY_PROBLEM when every observation is
// removed (errors.EmptyProblem, the reference raises the same).
extern "C" int ssfm_prune(int64_t n, const int32_t* cam_idx, const int32_t* pt_idx, int32_t C, int32_t P,
                          int32_t* camera_map, int32_t* point_map, uint8_t* obs_mask, int32_t* n_cam_out,
                          int32_t* n_pt_out, int64_t* n_obs_out, void* stream) {
  if (n < 0 || C < 0 || P < 0 || (n > 0 && (!cam_idx || !pt_idx)) || !camera_map || !point_map || !obs_mask)
    return set_err(SSFM_INVALID_ARGUMENT, "ssfm_prune: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  unsigned char *cam_ok = nullptr, *pt_ok = nullptr;
  int *cnt_cam = nullptr, *cnt_pt = nullptr, *scan = nullptr, *flag = nullptr, *changed = nullptr;
  unsigned long long* alive = nullptr;
  int *hchanged = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  const int M = std::max(C, P) + 1;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (int*)nullptr, (int*)nullptr, M, st);
  auto cleanup = [&]() {
    cudaFree(cam_ok); cudaFree(pt_ok); cudaFree(cnt_cam); cudaFree(cnt_pt); cudaFree(scan); cudaFree(flag);
    cudaFree(changed); cudaFree(alive); cudaFree(tmp);
    if (hchanged) cudaFreeHost(hchanged);
  };
  if (cudaMalloc(&cam_ok, C + 1) || cudaMalloc(&pt_ok, P + 1) || cudaMalloc(&cnt_cam, sizeof(int) * (C + 1)) ||
      cudaMalloc(&cnt_pt, sizeof(int) * (P + 1)) || cudaMalloc(&scan, sizeof(int) * M) ||
      cudaMalloc(&flag, sizeof(int) * M) || cudaMalloc(&changed, sizeof(int)) ||
      cudaMalloc(&alive, sizeof(unsigned long long)) || cudaMalloc(&tmp, tmp_bytes + 16) ||
      cudaMallocHost((void**)&hchanged, sizeof(int))) {
    cleanup();
    return set_err(SSFM_CUDA_ERROR, "ssfm_prune: out of memory");
  }
  cudaMemsetAsync(cam_ok, 1, C + 1, st);
  cudaMemsetAsync(pt_ok, 1, P + 1, st);
  cudaMemsetAsync(cnt_cam, 0, sizeof(int) * (C + 1), st);
  cudaMemsetAsync(cnt_pt, 0, sizeof(int) * (P + 1), st);
  const int gb = std::max(1, std::min(nblk(n, 256), 148 * 8));
  int rounds = 0;
  while (true) {   // the fixed point of ba.py:234-243
    cudaMemsetAsync(changed, 0, sizeof(int), st);
    if (n > 0) k_prune_count<<<gb, 256, 0, st>>>(cam_idx, pt_idx, n, cam_ok, pt_ok, cnt_cam, cnt_pt);
    if (P > 0) k_prune_drop<<<nblk(P, 256), 256, 0, st>>>(cnt_pt, pt_ok, P, 2, changed);
    if (C > 0) k_prune_drop<<<nblk(C, 256), 256, 0, st>>>(cnt_cam, cam_ok, C, 1, changed);
    cudaMemcpyAsync(hchanged, changed, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (cudaStreamSynchronize(st) != cudaSuccess) { cleanup(); return set_err(SSFM_CUDA_ERROR, "ssfm_prune"); }
    ++rounds;
    if (!*hchanged) break;
  }
  // maps: exclusive scans of the survivor flags
  int ncam = 0, npt = 0;
  auto make_map = [&](const unsigned char* ok, int cnt, int32_t* map, int* total) -> int {
    if (cnt == 0) { *total = 0; return 0; }
    k_prune_flags<<<nblk(cnt + 1, 256), 256, 0, st>>>(ok, cnt + 1, flag);
    cudaMemsetAsync(flag + cnt, 0, sizeof(int), st);
    size_t tb = tmp_bytes;
    if (cub::DeviceScan::ExclusiveSum(tmp, tb, flag, scan, cnt + 1, st)) return 1;
    k_prune_map<<<nblk(cnt, 256), 256, 0, st>>>(ok, scan, cnt, map);
    if (cudaMemcpyAsync(total, scan + cnt, sizeof(int), cudaMemcpyDeviceToHost, st)) return 1;
    return cudaStreamSynchronize(st) != cudaSuccess;
  };
  if (make_map(cam_ok, C, camera_map, &ncam) || make_map(pt_ok, P, point_map, &npt)) {
    cleanup();
    return set_err(SSFM_CUDA_ERROR, "ssfm_prune: map");
  }
  unsigned long long nalive = 0;
  cudaMemsetAsync(alive, 0, sizeof(unsigned long long), st);
  if (n > 0) k_prune_obs<<<gb, 256, 0, st>>>(cam_idx, pt_idx, n, cam_ok, pt_ok, obs_mask, alive);
  cudaMemcpyAsync(&nalive, alive, sizeof(nalive), cudaMemcpyDeviceToHost, st);
  const cudaError_t e = cudaStreamSynchronize(st);
  cleanup();
  if (e != cudaSuccess) return set_err(SSFM_CUDA_ERROR, std::string("ssfm_prune: ") + cudaGetErrorString(e));
  if (n_cam_out) *n_cam_out = ncam;
  if (n_pt_out) *n_pt_out = npt;
  if (n_obs_out) *n_obs_out = (int64_t)nalive;
  (void)rounds;
  if (nalive == 0) return set_err(SSFM_EMPTY_PROBLEM, "pruning removed every observation");
  return SSFM_OK;
}
