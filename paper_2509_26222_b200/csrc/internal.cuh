// Internal declarations of the B200 terralio library (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/terralio_gpu.h"

namespace tlg {

// ---------------------------------------------------------------------------
// Errors: internal code throws tlg::Error; every ABI entry point converts it
// into a status code + thread-local message (see guard() in abi.cu).
struct Error : std::runtime_error {
  tlg_status status;
  Error(tlg_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define TLG_CUDA(call)                                                       \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess) ::tlg::throw_cuda(_e, #call, __FILE__, __LINE__); \
  } while (0)

#define TLG_LAUNCHED(ctx)                                                    \
  do {                                                                       \
    cudaError_t _e = cudaPeekAtLastError();                                  \
    if (_e != cudaSuccess) ::tlg::throw_cuda(_e, "kernel launch", __FILE__, __LINE__); \
    ++(ctx)->launches;                                                       \
  } while (0)

struct NoSupported : Error {
  NoSupported() : Error(TLG_NO_SUPPORTED_CENTERS, "no supported centers") {}
};

inline void require(bool ok, tlg_status s, const char* msg) {
  if (!ok) throw Error(s, msg);
}

// ---------------------------------------------------------------------------
// Device buffers.
template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;    // capacity (elements)
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  // grow-only; contents are NOT preserved
  T* ensure(size_t count) {
    if (count <= n && p) return p;
    release();
    size_t c = count ? count : 1;
    cudaError_t e = cudaMalloc(&p, c * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      throw Error(e == cudaErrorMemoryAllocation ? TLG_OUT_OF_MEMORY : TLG_CUDA_ERROR,
                  std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    n = c;
    return p;
  }
  // grow preserving the first `keep` elements (stream-ordered copy)
  T* grow_keep(size_t count, size_t keep, cudaStream_t s) {
    if (count <= n && p) return p;
    DBuf nb;
    nb.ensure(count);
    if (keep && p) {
      cudaError_t e = cudaMemcpyAsync(nb.p, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) throw_cuda(e, "grow copy", __FILE__, __LINE__);
      cudaStreamSynchronize(s);
    }
    *this = std::move(nb);
    return p;
  }
};

// ---------------------------------------------------------------------------
// Scratch arena: named grow-only slots, reused across calls.
enum Slot : int {
  S_IN_X, S_IN_Y, S_IN_Z, S_IN_HX, S_IN_HY, S_IN_HZ,
  S_OUT_Z, S_OUT_GX, S_OUT_GY, S_OUT_SUP, S_OUT_R, S_OUT_J, S_OUT_RAW,
  S_FLAGS, S_PARTIALS, S_CUB, S_CUB2,
  S_KEYS, S_KEYS2, S_VALS, S_VALS2, S_NODES_X, S_NODES_Y, S_NODE_FLAG, S_NODE_IDX,
  S_COUNT, S_ACTIVE, S_BLOCKFLAG, S_ROWOF, S_MERGED, S_ROWPTR, S_COLIDX, S_MTVAL,
  S_KMAT, S_SMAT, S_RESID, S_U, S_YMAT, S_HMAT, S_WORK1, S_WORK2, S_WORK3, S_BLKTAB,
  S_MOMENT_ROW, S_TROWP, S_TKEYS, S_LINV, S_XINV, S_XINV2, S_SOLVE, S_BSOLVE, S_VALIDATE,
  S_GRAMPART, S_LATGRAM, S_LATSTART, S_LATPTS, S_LATNROW, S_FLOWFLAG, S_GEMVPART, S_REDSEG, S_FLOWORDER, S_GGPART,
  S_NUM_SLOTS
};

struct tlg_ctx_impl;

}  // namespace tlg

// ---------------------------------------------------------------------------
struct tlg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // H2D slices overlapping compute (manifold rows)
  cudaEvent_t copy_ev[9] = {};
  uint64_t launches = 0;
  int num_sms = 148;
  tlg::DBuf<unsigned char> slots[tlg::S_NUM_SLOTS];
  // pinned host staging
  void* pinned = nullptr;
  size_t pinned_bytes = 0;
  // hot-kernel profiling (tlg_ctx_set_profiling)
  bool profiling = false;
  cudaEvent_t prof_ev[2] = {nullptr, nullptr};
  double prof_ms[4] = {0, 0, 0, 0};
  uint64_t prof_n[4] = {0, 0, 0, 0};
  int prof_pending = -1;  // kernel id whose events await collection
  // dense.cu: inverses of the 64x64 diagonal Cholesky tiles of the most
  // recent potrf_lower (slot S_LINV), keyed by the factored matrix
  const double* linv_owner = nullptr;
  const double* linv32_owner = nullptr;  // factor whose 32-wide tile inverses S_LINV holds
  bool force_nb64 = false;  // dense_bench: force the 64-wide factorisation
  bool force_coop_potrf = false;  // diagnostics: the grid-barrier 32-wide factorisation
  long long flow_order_key = -1;   // (nt, bwt, skew) of the cached K7f claim order
  std::vector<int2> flow_order_host;  // its host copy (kept alive for the async upload)

  template <typename T>
  T* ws(int slot, size_t count) {
    // grow with 25 % headroom: per-scan sizes (n_active, m, nnz) fluctuate, and
    // every regrowth is a synchronising cudaFree/cudaMalloc pair
    size_t need = count * sizeof(T) + 16;
    if (need > slots[slot].n) need += need / 4;
    return reinterpret_cast<T*>(slots[slot].ensure(need));
  }
  void* host_stage(size_t bytes);
  void sync();
};

namespace tlg {

// Profiling brackets around one hot-kernel launch; prof_end() must be called
// after the stream has been synchronised.
void prof_begin(tlg_ctx* ctx, int kernel);
void prof_mark_end(tlg_ctx* ctx);
void prof_collect(tlg_ctx* ctx);

// Copy helpers honouring tlg_mem tags.
void copy_in(tlg_ctx* ctx, void* dst_dev, const void* src, size_t bytes, tlg_mem mem);
void copy_out(tlg_ctx* ctx, void* dst, const void* src_dev, size_t bytes, tlg_mem mem);
// Returns a device pointer holding `src` (no copy when already on device).
template <typename T>
const T* as_device(tlg_ctx* ctx, int slot, const T* src, size_t n, tlg_mem mem) {
  if (mem == TLG_DEVICE || n == 0) return src;
  T* d = ctx->ws<T>(slot, n);
  copy_in(ctx, d, src, n * sizeof(T), mem);
  return d;
}

// ---------------------------------------------------------------------------
// Exact (no-contraction) FP64 helpers: neighbour membership, lattice node
// coordinates and cell keys must round exactly like the reference's
// -O3/no-FMA host build.
__device__ __forceinline__ double sq2_exact(double dx, double dy) {
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// Kernel parameters after KernelParams::finalize, with derived constants.
struct KernelConst {
  double sigma, sigma_eps, lambda, cutoff;
  double r2;          // cutoff * cutoff (kernel.cpp:33, grid_index.hpp:36)
  double neg_inv_2s2; // -1 / (2 sigma^2)
  double neg_inv_2st2;// -1 / (2 sigma_tilde^2)
  double inv_s2;      // 1 / sigma^2 (terrain_model.cpp:129)
  double scale;       // moment_scale
  double sigma_tilde;
};
KernelConst make_kernel_const(const tlg_kernel_params& k);
void finalize_kernel(tlg_kernel_params& k);  // kernel.cpp:15-25

// Dense CSR grid over centre cells (GridIndex2 with cell = min(rho, 1e6)).
struct CenterGrid {
  double cell = 1.0;
  int span = 1;
  int gx0 = 0, gy0 = 0, gnx = 0, gny = 0;
  DBuf<int> cell_start;        // gnx*gny + 1
  DBuf<uint32_t> sorted_id;    // centre id in cell order (ids ascending inside a cell)
  DBuf<double> scx, scy, sw;   // centres/weights in cell order
};

struct GridView {
  const double* cx;
  const double* cy;
  const double* w;
  const uint32_t* id;
  const int* cell_start;
  double cell;
  int span, gx0, gy0, gnx, gny;
};

// Lattice fast path: when every centre is a mesh node roi.min + (i, j) * res
// (bit-exact, as select_centers / births produce them) and no node repeats,
// weights live in a dense zero-padded node grid W[i][j] and every query
// sweeps a fixed WIN x WIN node window whose pairs are pre-classified
// (always inside / boundary / always outside the cutoff disc).
constexpr int kMaxWin = 14;

// Window geometry for cutoff R (in lattice units): node offsets
// [-lo, win - lo) around the base cell; pair (k, l) is always inside the
// cutoff disc for every point of the (1e-6-expanded) base cell when
// dmax^2 < (R (1 - 1e-9))^2, and can never be when dmin^2 > (R (1 + 1e-9))^2.
// constexpr so the hot kernels can be specialised on it (eval.cu).
struct Geom {
  int win = 0, lo = 0;
  uint32_t in[16] = {0}, bd[16] = {0};
};

constexpr double geo_clamp(double v, double a, double b) { return v < a ? a : (v > b ? b : v); }
constexpr double geo_max(double a, double b) { return a > b ? a : b; }
constexpr double geo_abs(double a) { return a < 0 ? -a : a; }

constexpr Geom make_geom(double R) {
  Geom g{};
  const double mg = 1e-6;
  g.lo = static_cast<int>(R + mg);
  const int hi = static_cast<int>(1.0 + R + mg);
  g.win = g.lo + hi + 1;
  if (g.win > kMaxWin) {
    g.win = 0;
    return g;
  }
  const double rin = R * (1.0 - 1e-9), rout = R * (1.0 + 1e-9);
  for (int k = 0; k < g.win; ++k)
    for (int l = 0; l < g.win; ++l) {
      const double di = k - g.lo, dj = l - g.lo;
      const double nx = geo_clamp(di, -mg, 1.0 + mg), ny = geo_clamp(dj, -mg, 1.0 + mg);
      const double dmin2 = (di - nx) * (di - nx) + (dj - ny) * (dj - ny);
      const double fx = geo_max(geo_abs(di + mg), geo_abs(di - 1.0 - mg));
      const double fy = geo_max(geo_abs(dj + mg), geo_abs(dj - 1.0 - mg));
      const double dmax2 = fx * fx + fy * fy;
      if (dmax2 < rin * rin) g.in[k] |= 1u << l;
      else if (dmin2 <= rout * rout) g.bd[k] |= 1u << l;
    }
  return g;
}

// Geometries compiled into specialised kernels: the paper's parameters
// (sigma 0.04, sigma_eps 0.1 -> cutoff 0.32311 m, mesh 0.07 m; R = 4.6159)
// and the reference tests' (sigma 0.08, sigma_eps 0.05/0.02, mesh 0.12/0.1;
// R = 2.36..2.47). Any other R runs the runtime-mask kernel.
constexpr Geom kGeoms[] = {make_geom(4.615857142857142), make_geom(2.4)};
constexpr int kNumGeoms = 2;

inline bool geom_equal(const Geom& a, const Geom& b) {
  if (a.win != b.win || a.lo != b.lo) return false;
  for (int k = 0; k < 16; ++k)
    if (a.in[k] != b.in[k] || a.bd[k] != b.bd[k]) return false;
  return true;
}

struct __align__(16) AxisNode {
  double c;  // node coordinate min + k * res (reference rounding)
  int cell;  // floor(c / cell)
  int pad;
};

struct LatticeGrid {
  bool valid = false;
  int win = 0, lo = 0, pad = 0;
  int ni = 0, nj = 0;          // padded dims
  int i_org = 0, j_org = 0;    // lattice index of padded (0, 0)
  double org_x = 0, org_y = 0; // coordinate of padded node (0, 0) (for cell lookup only)
  double inv_res = 1;
  uint32_t inmask[16] = {0}, bdmask[16] = {0};
  int corner_ok = 0;
  int geom_id = -1;            // index into kGeoms when specialised, else -1
  DBuf<double> W;
  DBuf<double> W1;  // W shifted by one element (W1[s + 1] = W[s]): 16-byte pair loads at odd bases
  DBuf<int> P;                 // presence count per node
  DBuf<AxisNode> ax, ay;       // per padded column / row: exact node coordinate
                               // and reference cell coordinate floor(c / cell)
  // Cell-sweep ranges per point cell q: [first node with cell >= q - span,
  // first node with cell >= q + span + 1) along each axis (cells are monotone
  // in the node index), for q in [base, base + n) (clamped outside).
  DBuf<int2> xr, yr;
  // Per cell (ib, jb): LOOSE-path flags (k_cell_flags: bit 0 corner nodes
  // present, bit 1 skipped boundary tests provably negligible); rebuilt
  // lazily after weight syncs. pairlb: per window pair the minimum over the
  // cell of kappa and of kappa d (inside pairs; 0 otherwise).
  DBuf<uint8_t> cflag;
  DBuf<double> pairlb;
  bool wmax_dirty = true;
  int xr_base = 0, xr_n = 0, yr_base = 0, yr_n = 0;
  double min_x = 0, min_y = 0;  // node (i, j) = (min_x + (i + i_org) res, min_y + ...)
  DBuf<int> slot;              // centre id -> node index in W
};

struct LatticeView {
  const double* W;
  const double* W1;
  const int* P;
  const AxisNode* ax;  // one 16-byte load gives coordinate + cell
  const AxisNode* ay;
  const int2* xr;      // see LatticeGrid
  const int2* yr;
  const uint8_t* cflag;
  double loose_k;  // n_bd * kappa_sigma(cutoff)
  double loose_d;  // cutoff radius (gradient bound factor)
  int xr_base, xr_n, yr_base, yr_n, i_org, j_org;
  double min_x, min_y;
  int ni, nj, lo, span;
  double org_x, org_y, inv_res, cell;
  uint32_t inmask[16], bdmask[16];
  int corner_ok;
  int rec_ok;             // exp recurrence numerically safe for these parameters
  int loose_ok;           // beyond-cutoff boundary pairs negligible (eval.cu, LOOSE)
  double res, c_res, k2;  // lattice spacing, c*res, exp(2 c res^2) with c = -1/(2 s^2)
};

}  // namespace tlg

// ---------------------------------------------------------------------------
struct tlg_model {
  tlg_ctx* ctx = nullptr;
  tlg_kernel_params kernel{};
  tlg_center_params cparams{};
  tlg::KernelConst kc{};

  // Host mirror of the model *structure* (ids, blocks, tiles, occupancy),
  // the reference's bookkeeping in terrain_model.cpp:26-95.
  std::vector<double> hcx, hcy;
  std::vector<uint32_t> block_index;
  std::vector<std::vector<uint32_t>> members;
  std::unordered_map<int64_t, uint32_t> tile_blocks;
  std::unordered_set<int64_t> occupancy;

  // Device numeric state.
  tlg::DBuf<double> cx, cy, w;
  tlg::DBuf<uint32_t> d_block_index;
  size_t dev_cap = 0;
  // block info_inv pool: column-major, ld = blk_ld[b]
  tlg::DBuf<double> pool;
  size_t pool_used = 0;
  std::vector<size_t> blk_off;
  std::vector<int> blk_ld;
  tlg::CenterGrid grid;
  tlg::LatticeGrid lat;
  bool grid_dirty = true;
  bool exact_cutoff = false;  // force the per-pair cutoff test (tlg_model_set_exact_cutoff)
  bool batch_csr_gram = false;  // diagnostics: batch Gram by CSR rows even on a lattice
  int last_gram_lattice = 0;    // diagnostics: the last Gram assembly took the lattice path
  bool batch_block_order = false;  // diagnostics: batch-fit rows in block order even on a lattice
  // structural nonzeros of the banded batch system (positions in band
  // storage of centre pairs within 2 cutoffs): packs the partial systems of
  // the point-sharded fit for the cross-rank reduction; keyed by the centre
  // count it was built for
  tlg::DBuf<uint64_t> bpat;
  size_t bpat_nnz = 0, bpat_for = 0;
};

// A scan's lever arms, binned once per scan by the world cell they fall in
// under a reference pose, so LM cost evaluations read the weight grid with
// warp-coherent windows (tlg_scan_* in the ABI).
struct tlg_scan {
  tlg_ctx* ctx = nullptr;
  size_t n = 0;
  tlg::DBuf<double> hx, hy, hz;
  tlg::DBuf<uint32_t> perm;
  double bin_ms = 0.0;
};

namespace tlg {
int64_t pack2(int64_t x, int64_t y);
int64_t tile_key(const tlg_model* m, double cx, double cy);
int64_t mesh_node_key(const tlg_model* m, double x, double y);
uint32_t block_for_tile(tlg_model* m, int64_t key);

void build_center_grid(tlg_model* m);      // grid.cu
GridView grid_view(const tlg_model* m);    // grid.cu
LatticeView lattice_view(const tlg_model* m);
void ensure_grid(tlg_model* m);
int sweep_kind(const tlg_model* m);  // eval.cu
int prepare_sweep(tlg_model* m);     // sweep_kind + lazily built per-kind tables (grid.cu)
void sync_weights_to_grid(tlg_model* m);   // after weights change

// blocks / pool (model.cu)
void pool_reserve_block(tlg_model* m, uint32_t b, int new_size);

// select.cu: runs the support count over the lattice window; returns node
// count, writes nodes (device) into ctx slots S_NODES_X/Y. If occupancy_model
// is non-null, nodes already occupied in it are dropped (birth filter).
size_t supported_nodes_device(tlg_ctx* ctx, const double* dx, const double* dy, size_t m,
                              const tlg_center_params& p, const double** out_x,
                              const double** out_y);
void validate_obs_device(tlg_ctx* ctx, const double* x, const double* y, const double* z,
                         size_t m, size_t zn);
// Launch-only form: returns the device flag (read it at the next sync and
// pass it to validate_obs_check, which throws like validate_obs_device).
int* validate_obs_launch(tlg_ctx* ctx, const double* x, const double* y, const double* z,
                         size_t m, size_t zn);
void validate_obs_check(int flag);

// eval.cu
void eval_device(tlg_model* m, const double* x, const double* y, size_t n, double* z,
                 uint8_t* sup, double* gx, double* gy);
void manifold_device(tlg_model* m, const double R[9], const double t[3], const double* hx,
                     const double* hy, const double* hz, size_t n, double wheel_radius,
                     double lambda_M, double huber, double* r, double* J, uint8_t* valid,
                     double* raw, tlg_normal_eq* ne);

// update.cu
// pending_valid: flag of a validate_obs_launch not yet read; checked at the
// first synchronisation, before any state changes
void recursive_update_device(tlg_model* m, const double* x, const double* y, const double* z,
                             size_t mm, bool allow_birth, tlg_update_report* rep,
                             const int* pending_valid = nullptr);
void batch_fit_device(tlg_model* m, const double* x, const double* y, const double* z,
                      size_t mm);
void batch_system_dims(tlg_model* m, size_t* n, size_t* ld, size_t* elems);
void batch_assemble_device(tlg_model* m, const double* x, const double* y, const double* z,
                           size_t mm, double* H, size_t ld, double* b, bool add_lambda);
void batch_solve_device(tlg_model* m, double* H, size_t ld, double* b);
size_t batch_pattern_device(tlg_model* m);
// assemble.cu: lattice element assembly of the batch system (false: not a
// lattice / window too wide; nothing done)
bool lattice_gram_device(tlg_model* m, const double* x, const double* y, const double* z,
                         size_t mm, const int* rowof, int band, double* H, int ld, double* b);
void batch_pack_device(tlg_model* m, const double* H, double* packed);
void batch_unpack_device(tlg_model* m, const double* packed, double* H);

}  // namespace tlg
