// fht_api.cu -- C ABI (include/fht.h) and host dispatch for libfht.so.
//
// Host side: argument validation, frame geometry, the pass split m + L = K, batch
// chunking so one chunk's pass-1 scratch stays L2-resident, TMA tensor maps, and the launches.
// No device memory is allocated here; scratch and tables live in the caller's workspace.
//
// Two kernel generations share this dispatch:
//   v2 (fht_tile.cuh) -- register-resident warp butterflies + TMA stores; every frame with
//                        K >= 2 and at least 8 columns in both passes (all BASELINE configs).
//   v1 (fht_kernels.cuh) -- level-by-level shared-memory butterflies; only the degenerate
//                        frames v2 does not tile (Hp <= 2 or fewer than 8 columns).
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <utility>

#include "../../include/fht.h"
#include "fht_kernels.cuh"
#include "fht_tile.cuh"
#include "fht_p1p.cuh"
#include "fht_p1p8.cuh"
#include "fht_internal.cuh"
#include "fht_peaks.cuh"

namespace {

using namespace fht;
using namespace fht::detail;

// Pass-1 scratch bytes per batch chunk. Measured (profiles/r01_v2/ab_scratch_budget*.log): fewer, fuller
// launches beat keeping a chunk's scratch L2-resident -- C5 1528 us at 48 MiB (1 image per chunk),
// 1391 us with the whole 16-image batch (1.1 GB) in one chunk; C3 318 -> 302 us. 2 GiB of a B200's
// 180 GB (two buffers when a batch needs several chunks).
#ifndef FHT_SCRATCH_BUDGET_MB
#define FHT_SCRATCH_BUDGET_MB 2048
#endif
// (the environment variable FHT_SCRATCH_BUDGET_MB overrides it: tests of the multi-chunk schedule)
size_t scratch_budget() {
  const char* e = std::getenv("FHT_SCRATCH_BUDGET_MB");
  const long mb = e ? std::atol(e) : 0;
  return size_t(mb > 0 ? mb : FHT_SCRATCH_BUDGET_MB) << 20;
}

int64_t next_pow2(int64_t n) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  return p;
}
int ilog2(int64_t p) {
  int k = 0;
  while ((int64_t(1) << k) < p) ++k;
  return k;
}
size_t dtype_size(int dt) { return dt == FHT_U8 ? 1 : 4; }
int out_dtype(int in_dt) { return in_dt == FHT_F32 ? FHT_F32 : FHT_I32; }
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// Frame of one orientation (mostly-horizontal quadrants use the transposed image).
struct Frame {
  int transposed;
  int Hp, K;        // FHT rows (power of two), K = log2 Hp
  int wc;           // content width (columns that may hold pixels: image cols, or Wp in FULL)
  int W;            // cyclic width wc + Hp
  int rows_avail;   // FHT rows actually backed by the image
  int cols_avail;   // FHT columns actually backed by the image
  int m, L;         // pass split
};

// Pass split K = m + L (both <= 6). 32-row pass-2 tiles (L = 5) are the most efficient measured
// (C3, K = 9: 4 + 5 beats 5 + 4 by 15%); 64-row tiles (6) are the least (C5, K = 11: 6 + 5 beats
// 5 + 6 by 15%), so pass 2 gets min(5, ceil(K/2)) levels unless pass 1 would exceed 6.
void split_levels(Frame& f) {
  const int half_up = (f.K + 1) / 2;
  f.L = f.K - 6 > (half_up < 5 ? half_up : 5) ? f.K - 6 : (half_up < 5 ? half_up : 5);
  if (f.L > f.K) f.L = f.K;
  if (const int l = env_int("FHT_SPLIT_L", 0)) {  // A/B: pass-2 levels (both passes must stay <= 6)
    if (l <= 6 && f.K - l <= 6 && l < f.K) f.L = l;
  }
  f.m = f.K - f.L;
  if (f.m < 1 && f.K >= 2) {  // keep pass 1 non-empty
    f.m = 1;
    f.L = f.K - 1;
  }
  if (f.K <= 1) {  // Hp <= 2: one pass-1 level (v1 path)
    f.m = f.K;
    f.L = 0;
  }
}

Frame make_frame(int64_t h, int64_t w, int transposed, int full, int64_t pad = -1) {
  Frame f{};
  f.transposed = transposed;
  const int64_t rows = transposed ? w : h, cols = transposed ? h : w;
  f.Hp = (int)next_pow2(rows);
  f.K = ilog2(f.Hp);
  f.wc = full ? (int)next_pow2(cols) : (int)cols;  // R9: FULL pads both dims to powers of two
  f.W = f.wc + (pad < 0 ? f.Hp : (int)pad);          // extended by pad (default Hp) columns
  f.rows_avail = (int)rows;
  f.cols_avail = (int)cols;
  split_levels(f);
  return f;
}

int check_image(const fht_image* img) {
  if (!img || !img->data) return FHT_ERR_ARG;
  if (img->dtype != FHT_U8 && img->dtype != FHT_I32 && img->dtype != FHT_F32) return FHT_ERR_DTYPE;
  if (img->batch < 1 || img->h < 1 || img->w < 1) return FHT_ERR_ARG;
  if (img->row_stride < img->w || (img->batch > 1 && img->batch_stride < img->h * img->row_stride))
    return FHT_ERR_ARG;
  if (img->h > (1 << 20) || img->w > (1 << 20)) return FHT_ERR_UNSUPPORTED;
  const size_t es = dtype_size(img->dtype);
  if ((reinterpret_cast<uintptr_t>(img->data) % es) != 0) return FHT_ERR_ALIGN;
  return FHT_OK;
}

int check_frame_supported(const Frame& f) {
  if (f.m > kMaxLog || f.L > kMaxLog) return FHT_ERR_UNSUPPORTED;  // Hp > 4096 needs 3 passes
  if ((int64_t)f.W + 2 * f.Hp > (int64_t(1) << 30)) return FHT_ERR_UNSUPPORTED;
  return FHT_OK;
}

// ---------------------------------------------------------------- pass geometry (v1 and v2)
// Pass-1 range of F_m for a slot: sigma=+1 [-(2^m-1), wc), sigma=-1 [0, wc + 2^m - 1); range mode
// uses the plan's shear extent.
struct RangeDev {
  const int* e_tab;
  const int* colmap;
  const int* start_tab;
  const int* len_tab;
  double alpha;               // §4 scale: >= 1 lets pass 1 load image rows by TMA (dilation)
  int transposed;             // mostly-horizontal plan: frame rows are image columns (gather fill)
  int rows;                   // output rows (plan.rows; < Hp for a pruned plan, f2)
  int w_content, x_lo, x_hi;  // scratch signed x range (pass 1)
  int out_lo, out_hi;         // signed x range covered by pass 2 tiles
};

void pass1_range(const Frame& f, int sigma, const RangeDev* rg, int& lo, int& hi) {
  if (rg) { lo = rg->x_lo; hi = rg->x_hi; return; }
  const int hm = (1 << f.m) - 1;
  lo = sigma > 0 ? -hm : 0;
  hi = sigma > 0 ? f.wc : f.wc + hm;
}

bool use_v2(const Frame& f, const RangeDev* rg) {
  if (f.K < 2 || f.m > 6 || f.L < 1 || f.L > 6) return false;
  int lo, hi;
  pass1_range(f, +1, rg, lo, hi);
  if (hi - lo < 8) return false;
  pass1_range(f, -1, rg, lo, hi);
  if (hi - lo < 8) return false;
  const int span2 = rg ? rg->out_hi - rg->out_lo : f.W;
  return f.W >= 12 && span2 >= 12;
}

// v2 pass-1 columns [lo, hi) rounded up to a multiple of 4 (16-byte aligned TMA rows); the
// extra columns hold zeros (no pixel reaches them), so pass 2 may read them freely.
// pass-1 scratch element bytes: u8 input keeps F_m in uint16, else the accumulator
int scratch_es(int dtype) { return dtype == FHT_U8 ? 2 : 4; }
// spans rounded to 16 bytes of scratch elements (tile starts and row pitch stay TMA-aligned)
void v2_pass1_range(const Frame& f, int sigma, const RangeDev* rg, int& lo, int& hi, int es) {
  pass1_range(f, sigma, rg, lo, hi);
  // the span is a multiple of 32 columns (FHT_ROW32: pass 2 reads the scratch as [row][col/32][32]); the
  // columns added past the support are computed by pass 1 as exact zeros
  const int al = FHT_ROW32 ? 32 : 16 / es;
  hi = lo + ((hi - lo + al - 1) & ~(al - 1));
}
int64_t v2_scratch_pitch(const Frame& f, const RangeDev* rg, int es) {
  int lo, hi, w = 0;
  for (int s = -1; s <= 1; s += 2) {
    v2_pass1_range(f, s, rg, lo, hi, es);
    w = (hi - lo) > w ? (hi - lo) : w;
  }
  return w;
}

// v1 scratch
int v1_scratch_width(const Frame& f) {
  const int ws = f.wc + (1 << f.m) - 1;
  return (ws + 3) & ~3;
}

// at most kMaxChunk images per launch: the v1 grid puts image x slot in gridDim.z (<= 65535, 4 slots)
// and the v2 flat grids stay below 2^31 CTAs
constexpr int64_t kMaxChunk = 16383;
int chunk_images(size_t per_image_touched, int64_t batch) {
  int64_t c = (int64_t)(scratch_budget() / (per_image_touched ? per_image_touched : 1));
  if (c < 1) c = 1;
  if (c > kMaxChunk) c = kMaxChunk;
  if (c > batch) c = batch;
  const int64_t n = (batch + c - 1) / c;  // balanced: 17 images at most 16 per chunk -> 9 + 8
  return (int)((batch + n - 1) / n);
}

// Scratch bytes (address extent) and chunk for one orientation with nq slots.
struct ScratchPlan {
  int v2;
  int64_t pitch;       // elements
  int chunk;
  int nbuf;            // scratch buffers: 2 when the batch needs several chunks (pass overlap)
  size_t bytes;        // all buffers
};
ScratchPlan scratch_plan(const Frame& f, int nq, int64_t batch, const RangeDev* rg, int es) {
  ScratchPlan sp{};
  sp.v2 = use_v2(f, rg);
  if (sp.v2) {
    sp.pitch = v2_scratch_pitch(f, rg, es);
    const size_t touched = (size_t)nq * f.Hp * (size_t)sp.pitch * es;
    sp.chunk = rg ? 1 : chunk_images(touched, batch);
    sp.nbuf = batch > sp.chunk ? 2 : 1;
    sp.bytes = (size_t)sp.nbuf * sp.chunk * nq * f.Hp * (size_t)sp.pitch * es;
  } else {
    sp.nbuf = 1;
    sp.pitch = rg ? ((rg->x_hi - rg->x_lo + 3) & ~3) : v1_scratch_width(f);
    const size_t per = (size_t)nq * f.Hp * (size_t)sp.pitch * 4;
    sp.chunk = rg ? 1 : chunk_images(per, batch);
    sp.bytes = per * sp.chunk;
  }
  return sp;
}

// ---------------------------------------------------------------- pipelined passes (fht_pipe.cuh)
// One persistent kernel for both passes over units of (nbu images, one slot), NBUF ring buffers of
// scratch (L2-resident), pass 1 of unit u + D beside pass 2 of unit u. Used for non-range v2 frames
// with Hp in [256, 4096] and at least two units; FHT_PIPE=1 opts in (measured slower than the two-launch path: DESIGN.md §5).
bool pipe_split_ok(int m, int L) {
  return (m == 4 && L == 4) || (m == 4 && L == 5) || (m == 5 && L == 5) || (m == 6 && L == 5) || (m == 6 && L == 6);
}
struct PipePlan {
  int on;
  int nbu, D, NBUF, nunits;
  int64_t pitch;
  size_t scratch_bytes;  // ring (256-byte rounded); the counters follow
  size_t bytes;          // ring + counters
};
PipePlan pipe_plan(const Frame& f, int nq, int64_t batch, const RangeDev* rg, int es) {
  PipePlan pp{};
  // (the pipelined kernel's persistent mbarriers need the per-warp loads: FHT_P1/P2_WARPLOAD)
  if (!(FHT_P1_WARPLOAD && FHT_P2_WARPLOAD) || rg || !use_v2(f, rg) || !pipe_split_ok(f.m, f.L) ||
      env_int("FHT_PIPE", 0) == 0)
    return pp;  // opt-in (measured slower)
  pp.pitch = v2_scratch_pitch(f, rg, es);
  const size_t per = (size_t)f.Hp * (size_t)pp.pitch * es;  // one image, one slot
  const size_t target = (size_t)env_int("FHT_PIPE_UNIT_MB", 16) << 20;
  int64_t nbu = (int64_t)(target / per);
  if (nbu < 1) nbu = 1;
  if (nbu > batch) nbu = batch;
  while (batch % nbu) --nbu;  // units of equal size
  const int64_t nunits = (batch / nbu) * nq;
  if (nunits < 2 || nunits > (1 << 20)) return pp;
  pp.nbu = (int)nbu;
  pp.nunits = (int)nunits;
  pp.D = env_int("FHT_PIPE_D", 2);
  if (pp.D < 1) pp.D = 1;
  if (pp.D > pp.nunits) pp.D = pp.nunits;
  pp.NBUF = env_int("FHT_PIPE_NBUF", pp.D + 2);
  if (pp.NBUF < pp.D + 1) pp.NBUF = pp.D + 1;
  if (pp.NBUF > pp.nunits) pp.NBUF = pp.nunits;
  pp.scratch_bytes = ((size_t)pp.NBUF * nbu * per + 255) & ~size_t(255);
  pp.bytes = pp.scratch_bytes + (size_t)(1 + 2 * nunits) * sizeof(int);
  pp.on = 1;
  return pp;
}

// ---------------------------------------------------------------- TMA tensor maps
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 2-D row-major tensor [rows][cols] with a box_rows x box_cols box (default: one row per copy).
bool make_row_map(CUtensorMap* m, const void* base, bool f32, uint64_t cols, uint64_t rows, uint64_t pitch_elems,
                  uint32_t box_cols, uint32_t box_rows = 1, bool u16 = false) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_elems * (u16 ? 2 : 4)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  const CUtensorMapDataType dt = u16 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                     : f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_INT32;
  return fn(m, dt, 2, const_cast<void*>(base), dims,
            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Pass-2 scratch reads: FHT_ROW32 -- the view [rows][cols/32][32] (cols = the pass-1 span, a multiple of 32), box
// {32, 10, 1} = one 320-column row per copy (scr1 unused); else 2-D rows, boxes of 256 and 36 (u16: 40) columns.
bool make_scr_maps(CUtensorMap* m0, CUtensorMap* m1, const void* base, bool f32, bool u16, uint64_t cols,
                   uint64_t rows, uint64_t pitch_elems) {
#if FHT_ROW32
  auto fn = encode_fn();
  if (!fn || cols % 32 != 0) return false;
  const uint64_t es = u16 ? 2 : 4;
  cuuint64_t dims[3] = {32, cols / 32, rows};
  cuuint64_t strides[2] = {32 * es, pitch_elems * es};
  cuuint32_t box[3] = {32, 10, 1};
  cuuint32_t e[3] = {1, 1, 1};
  const CUtensorMapDataType dt = u16 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                     : f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_INT32;
  if (fn(m0, dt, 3, const_cast<void*>(base), dims, strides, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  *m1 = *m0;
  return true;
#else
  return make_row_map(m0, base, f32, cols, rows, pitch_elems, 256, 1, u16) &&
         make_row_map(m1, base, f32, cols, rows, pitch_elems, u16 ? 40 : 36, 1, u16);
#endif
}

// ---------------------------------------------------------------- v1 launch helpers
template <typename Tin, int LOGR>
cudaError_t launch_pass1_t(dim3 grid, const Pass1Args& a, cudaStream_t st) {
  using A = typename AccOf<Tin>::type;
  constexpr int R = 1 << LOGR;
  const size_t smem = 2 * (size_t)R * tile_pitch(R) * sizeof(A);
  static std::atomic<unsigned long long> done{0};
  const cudaError_t attr = smem_optin(k_pass1<Tin, LOGR>, smem, done);
  if (attr != cudaSuccess) return attr;
  k_pass1<Tin, LOGR><<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename Tin>
cudaError_t launch_pass1(int logr, dim3 grid, const Pass1Args& a, cudaStream_t st) {
  switch (logr) {
    case 0: return launch_pass1_t<Tin, 0>(grid, a, st);
    case 1: return launch_pass1_t<Tin, 1>(grid, a, st);
    case 2: return launch_pass1_t<Tin, 2>(grid, a, st);
    case 3: return launch_pass1_t<Tin, 3>(grid, a, st);
    case 4: return launch_pass1_t<Tin, 4>(grid, a, st);
    case 5: return launch_pass1_t<Tin, 5>(grid, a, st);
    case 6: return launch_pass1_t<Tin, 6>(grid, a, st);
  }
  return cudaErrorInvalidValue;
}

template <typename A, int LOGR>
cudaError_t launch_pass2_t(dim3 grid, const Pass2Args& a, cudaStream_t st) {
  constexpr int R = 1 << LOGR;
  const size_t smem = 2 * (size_t)R * tile_pitch(R) * sizeof(A);
  static std::atomic<unsigned long long> done{0};
  const cudaError_t attr = smem_optin(k_pass2<A, LOGR>, smem, done);
  if (attr != cudaSuccess) return attr;
  k_pass2<A, LOGR><<<grid, kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename A>
cudaError_t launch_pass2(int logr, dim3 grid, const Pass2Args& a, cudaStream_t st) {
  switch (logr) {
    case 0: return launch_pass2_t<A, 0>(grid, a, st);
    case 1: return launch_pass2_t<A, 1>(grid, a, st);
    case 2: return launch_pass2_t<A, 2>(grid, a, st);
    case 3: return launch_pass2_t<A, 3>(grid, a, st);
    case 4: return launch_pass2_t<A, 4>(grid, a, st);
    case 5: return launch_pass2_t<A, 5>(grid, a, st);
    case 6: return launch_pass2_t<A, 6>(grid, a, st);
  }
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------- v2 launch helpers
struct P1Maps {
  CUtensorMap img0, img1;
  v2::P1Dst dst;
  CUtensorMap imgT;  // u8 transposed tiles (v2::P1Params::tfill_tma), else a copy of img0 (unused)
  CUtensorMap img8, imgS, dst4;  // persistent pass 1 (k_p1p): image box {32, 10, 8, 1}, swizzled image box
                                 // {32, 144, 1} (transposed slots), scratch box {TX, 1, 4, 1}
  int persist = 0;         // launch k_p1p instead of k_p1
  void* scr = nullptr;     // k_p1p: the scratch buffer [z][j][strip][pitch] and its row pitch (elements)
  int64_t scr_pitch = 0;
};

// Pass-1 destination view [z][j][strip][column] of a scratch buffer (dims column, strip, j, z; S strips,
// J shifts, Z images x slots), box {TX, 1, jper, 1}: one tile's shifts j of one destination.
bool make_dst_map(CUtensorMap* m, void* base, int ses, bool f32, int64_t pitch, int64_t S, int64_t J, int64_t Z, int TX,
                  int jper) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t rb = (cuuint64_t)(pitch * ses);
  cuuint64_t dims[4] = {(cuuint64_t)pitch, (cuuint64_t)S, (cuuint64_t)J, (cuuint64_t)Z};
  cuuint64_t strides[3] = {rb, rb * (cuuint64_t)S, rb * (cuuint64_t)(S * J)};
  cuuint32_t box[4] = {(cuuint32_t)TX, 1, (cuuint32_t)jper, 1};
  cuuint32_t e[4] = {1, 1, 1, 1};
  const CUtensorMapDataType sdt = ses == 2 ? CU_TENSOR_MAP_DATA_TYPE_UINT16
                                           : f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_INT32;
  return fn(m, sdt, 4, base, dims, strides, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
template <typename Tin, int R>
cudaError_t launch_p1_t(dim3 grid, const P1Maps& m, const v2::P1Params& a, cudaStream_t st) {
  // range launches with the TMA loader also stage the strip's colmap slice (kColmapStageBytes)
  const size_t smem = v2::p1_smem_bytes(R, sizeof(Tin) == 1) + (a.range && a.fill_tma ? v2::kColmapStageBytes : 0);
  static std::atomic<unsigned long long> done{0};
  const cudaError_t attr =
      smem_optin(v2::k_p1<Tin, R>, v2::p1_smem_bytes(R, sizeof(Tin) == 1) + v2::kColmapStageBytes, done);
  if (attr != cudaSuccess) return attr;
  return launch_pdl(v2::k_p1<Tin, R>, grid, dim3(v2::Split<R>::nw * 32), smem, st, m.img0, m.img1, m.dst, a, m.imgT);
}
// Persistent pass 1 (fht_p1p.cuh): 64-row strips of 4-byte images, all 64 shifts to one scratch; two CTAs per SM
// walk the tiles of `grid` (the k_p1 grid of the same launch), gridDim.x a multiple of the slot count.
template <typename Tin>
cudaError_t launch_p1p_t(dim3 grid, const P1Maps& m, const v2::P1Params& a, cudaStream_t st) {
  const size_t smem = v2::p1p_smem_bytes(a.range != 0);
  static std::atomic<unsigned long long> done{0};
  cudaError_t e = smem_optin(v2::k_p1p<Tin>, v2::p1p_smem_bytes(true), done);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess ||
      (e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
    return e;
  const long long total = (long long)grid.x * grid.y * grid.z;
  if (total <= 0 || total >= (1ll << 31) - 4096) return cudaErrorInvalidValue;
  long long G = 2ll * nsm;
  G -= G % a.nq;
  if (G < a.nq) G = a.nq;
  if (G > total) G = total;
  return launch_pdl(v2::k_p1p<Tin>, dim3((unsigned)G), dim3(256), smem, st, m.img8, m.imgS, m.dst4, a, (int)total, m.scr,
                    m.scr_pitch);
}
// Persistent pass 1 for 16-row strips of u8 images (fht_p1p8.cuh): six 4-warp CTAs per SM.
inline cudaError_t launch_p1p8(dim3 grid, const P1Maps& m, const v2::P1Params& a, cudaStream_t st) {
  const size_t smem = v2::p1p8_smem_bytes();
  static std::atomic<unsigned long long> done{0};
  cudaError_t e = smem_optin(v2::k_p1p8, smem, done);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess ||
      (e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
    return e;
  const long long total = (long long)grid.x * grid.y * grid.z;
  if (total <= 0 || total >= (1ll << 31) - 4096) return cudaErrorInvalidValue;
  long long G = (long long)env_int("FHT_P1P8_CTAS", 6) * nsm;  // CTAs per SM (A/B; 6 fit: 36 KB each)
  G -= G % a.nq;
  if (G < a.nq) G = a.nq;
  if (G > total) G = total;
  return launch_pdl(v2::k_p1p8, dim3((unsigned)G), dim3(128), smem, st, m.img8, m.imgT, m.dst4, a, (int)total);
}
template <typename Tin>
cudaError_t launch_p1(int r, dim3 grid, const P1Maps& m, const v2::P1Params& a, cudaStream_t st) {
  if constexpr (sizeof(Tin) == 4) {
    if (m.persist && r == 6) return launch_p1p_t<Tin>(grid, m, a, st);
  }
  if constexpr (sizeof(Tin) == 1) {
    if (m.persist && r == 4) return launch_p1p8(grid, m, a, st);
  }
  switch (r) {
    case 1: return launch_p1_t<Tin, 1>(grid, m, a, st);
    case 2: return launch_p1_t<Tin, 2>(grid, m, a, st);
    case 3: return launch_p1_t<Tin, 3>(grid, m, a, st);
    case 4: return launch_p1_t<Tin, 4>(grid, m, a, st);
    case 5: return launch_p1_t<Tin, 5>(grid, m, a, st);
    case 6: return launch_p1_t<Tin, 6>(grid, m, a, st);
  }
  return cudaErrorInvalidValue;
}
struct P2Maps {
  CUtensorMap scr0, scr1, out0, out1, out0_box;
};
template <typename A, int R, typename Tscr>
cudaError_t launch_p2_t(dim3 grid, const P2Maps& m, const v2::P2Params& a, cudaStream_t st) {
  const size_t smem = v2::p2_smem_bytes(R);
  static std::atomic<unsigned long long> done{0};
  const cudaError_t attr = smem_optin(v2::k_p2<A, R, Tscr>, smem, done);
  if (attr != cudaSuccess) return attr;
  return launch_pdl(v2::k_p2<A, R, Tscr>, grid, dim3(v2::Split<R>::nw * 32), smem, st, m.scr0, m.scr1, m.out0, m.out1,
                    m.out0_box, a);
}
template <typename A, typename Tscr = A>
cudaError_t launch_p2(int r, dim3 grid, const P2Maps& m, const v2::P2Params& a, cudaStream_t st) {
  switch (r) {
    case 1: return launch_p2_t<A, 1, Tscr>(grid, m, a, st);
    case 2: return launch_p2_t<A, 2, Tscr>(grid, m, a, st);
    case 3: return launch_p2_t<A, 3, Tscr>(grid, m, a, st);
    case 4: return launch_p2_t<A, 4, Tscr>(grid, m, a, st);
    case 5: return launch_p2_t<A, 5, Tscr>(grid, m, a, st);
    case 6: return launch_p2_t<A, 6, Tscr>(grid, m, a, st);
  }
  return cudaErrorInvalidValue;
}

// 3-D image tensor [batch][h][w] (elements of 1 or 4 bytes), box 1 x 1 x box_cols.
bool make_image_map(CUtensorMap* m, const fht_image* img, uint32_t box_cols) {
  auto fn = encode_fn();
  if (!fn) return false;
  const uint64_t es = dtype_size(img->dtype);
  cuuint64_t dims[3] = {(cuuint64_t)img->w, (cuuint64_t)img->h, (cuuint64_t)img->batch};
  cuuint64_t strides[2] = {(cuuint64_t)(img->row_stride * es), (cuuint64_t)(img->batch_stride * es)};
  if (img->batch == 1) strides[1] = (cuuint64_t)(img->h * img->row_stride * es);
  cuuint32_t box[3] = {box_cols, 1, 1};
  cuuint32_t e[3] = {1, 1, 1};
  const CUtensorMapDataType dt = img->dtype == FHT_U8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                 : img->dtype == FHT_I32 ? CU_TENSOR_MAP_DATA_TYPE_INT32
                                                         : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  return fn(m, dt, 3, const_cast<void*>(img->data), dims, strides, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

// Pass-1 fill32 (FHT_ROW32, 4-byte images with w % 32 == 0): the view [img][row][col/32][32], box {32, 10, 1, 1}
// = one 320-column row per copy from a 128-byte aligned column.
bool make_image_map32(CUtensorMap* m, const fht_image* img, uint32_t box_rows = 1) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {32, (cuuint64_t)(img->w / 32), (cuuint64_t)img->h, (cuuint64_t)img->batch};
  cuuint64_t strides[3] = {128, (cuuint64_t)(img->row_stride * 4), (cuuint64_t)(img->batch_stride * 4)};
  if (img->batch == 1) strides[2] = (cuuint64_t)(img->h * img->row_stride * 4);
  cuuint32_t box[4] = {32, 10, box_rows, 1};
  cuuint32_t e[4] = {1, 1, 1, 1};
  const CUtensorMapDataType dt = img->dtype == FHT_I32 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  return fn(m, dt, 4, const_cast<void*>(img->data), dims, strides, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}
// Persistent u8 pass 1 (k_p1p8): the view [img][row][col/128][128] bytes, box {128, 4, 4 rows, 1}: one copy of 4
// rows x 512 columns from a 128-byte aligned column (w % 128 == 0).
bool make_image_map128(CUtensorMap* m, const fht_image* img) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {128, (cuuint64_t)(img->w / 128), (cuuint64_t)img->h, (cuuint64_t)img->batch};
  cuuint64_t strides[3] = {128, (cuuint64_t)img->row_stride, (cuuint64_t)img->batch_stride};
  if (img->batch == 1) strides[2] = (cuuint64_t)(img->h * img->row_stride);
  cuuint32_t box[4] = {128, 4, 4, 1};
  cuuint32_t e[4] = {1, 1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(img->data), dims, strides, box, e,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// Persistent pass 1, transposed slots (k_p1p): the 4-byte image [img][row][col], box {32 columns, 144 rows, 1} with
// the 128-byte swizzle (16-byte chunk ^ (row & 7)): the block lands untransposed and is read column-wise without
// bank conflicts.
bool make_image_map_swz(CUtensorMap* m, const fht_image* img) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)img->w, (cuuint64_t)img->h, (cuuint64_t)img->batch};
  cuuint64_t strides[2] = {(cuuint64_t)(img->row_stride * 4), (cuuint64_t)(img->batch_stride * 4)};
  if (img->batch == 1) strides[1] = (cuuint64_t)(img->h * img->row_stride * 4);
  cuuint32_t box[3] = {32, (cuuint32_t)v2::kP1pBoxRows, 1};
  cuuint32_t e[3] = {1, 1, 1};
  const CUtensorMapDataType dt = img->dtype == FHT_I32 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  return fn(m, dt, 3, const_cast<void*>(img->data), dims, strides, box, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}
// u8 transposed pass-1 tiles (v2::P1Params::tfill_tma): the image [img][row][col] bytes, box {2^R columns, 144 rows}
bool make_imgT_map(P1Maps& m, v2::P1Params& p1, const fht_image* img, int R) {
  p1.tfill_tma = 0;
  m.imgT = m.img0;
  if (img->dtype != FHT_U8 || R < 4 || p1.range || !aligned16(img->data) || img->row_stride % 16 != 0 ||
      (img->batch > 1 && img->batch_stride % 16 != 0) || env_int("FHT_TFILL_TMA", 1) == 0)
    return true;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)img->w, (cuuint64_t)img->h, (cuuint64_t)img->batch};
  cuuint64_t strides[2] = {(cuuint64_t)img->row_stride,
                           (cuuint64_t)(img->batch == 1 ? img->h * img->row_stride : img->batch_stride)};
  cuuint32_t box[3] = {(cuuint32_t)(1 << R), 144, 1};
  cuuint32_t e[3] = {1, 1, 1};
  if (fn(&m.imgT, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(img->data), dims, strides, box, e,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  p1.tfill_tma = 1;
  return true;
}
bool make_p1_image_maps(CUtensorMap* m0, CUtensorMap* m1, const fht_image* img, const v2::P1Params& p1, size_t es) {
  if (p1.fill32) {
    if (!make_image_map32(m0, img)) return false;
    *m1 = *m0;
    return true;
  }
  return make_image_map(m0, img, 256) && make_image_map(m1, img, es == 1 ? 48 : 36);
}

// One quadrant slot: sign, source orientation and output row placement.
struct Slot {
  int sigma;
  int transposed;
  int64_t qrow;          // output row (in the [batch*rows_per_img][W] view) of the quadrant's row 0
  int row_base, row_sign, skip_t;
};

// Output destinations: [0] = Hough image, [1] = its fhtshift (either may be NULL).
struct Outs {
  const fht_hough* d[2];
};

// Launch accounting across one ABI call: counts kernels and records the caller's optional
// timing events (fht_exec_opts) before launch i and after the last launch.
struct LaunchLog {
  const fht_exec_opts* opts;
  int n;
  cudaEvent_t mark_first = nullptr;  // recorded after the first launch (the staggered orientation split)
  void before(cudaStream_t st) {
    if (opts && opts->events && n < opts->n_events) cudaEventRecord((cudaEvent_t)opts->events[n], st);
  }
  void after(cudaStream_t st) {
    ++n;
    if (opts && opts->events && n < opts->n_events) cudaEventRecord((cudaEvent_t)opts->events[n], st);
    if (mark_first && n == 1) cudaEventRecord(mark_first, st);
  }
};

// One phase of a sharded transform (fht_shard_*): phase 1 runs pass 1 on this rank's
// strips into the world destinations dst[h]; phase 2 runs pass 2 on this rank's groups from `recv`.
struct ShardCfg {
  int world, rank, phase;
  int64_t S, J;          // strips and groups per rank (2^L / world, 2^m / world)
  void* const* dst;      // phase 1: dst[h] = where rank h's chunk goes
  const void* recv;      // phase 2: [world][z][j_local][strip_local][pitch]
  int64_t chunk_rows;    // z * J * S
};

// Run the two passes for one orientation over all images, chunked (or one phase of a shard). Returns
// launches or error.
int run_orientation(const fht_image* img, const Frame& f, const Slot* slots, int nq, const Outs& outs, void* ws,
                    size_t ws_bytes, cudaStream_t st, const RangeDev* rg, LaunchLog& log,
                    const ShardCfg* sh = nullptr) {
  const int ses = scratch_es(img->dtype);
  const ScratchPlan sp = scratch_plan(f, nq, img->batch, rg, ses);
  const PipePlan pq = sh ? PipePlan{} : pipe_plan(f, nq, img->batch, rg, ses);
  const bool pipe = pq.on && ws && ws_bytes >= pq.bytes;
  if (!sh && (!ws || (ws_bytes < sp.bytes && !pipe))) return FHT_ERR_WORKSPACE;
  if (sh && !sp.v2) return FHT_ERR_UNSUPPORTED;
  int launches = 0;
  const fht_hough* any = outs.d[0] ? outs.d[0] : outs.d[1];

  if (sp.v2) {
    const int nstrips = 1 << f.L;
    // pass-2 groups j = rows t >> L: a pruned range plan (f2) needs only t < rows
    const int ngroups = rg && rg->rows < f.Hp ? (rg->rows + nstrips - 1) / nstrips : 1 << f.m;
    const size_t es = dtype_size(img->dtype);
    v2::P1Params p1{};
    p1.img = img->data;
    p1.img_bstride = img->batch_stride;
    p1.img_rstride = img->row_stride;
    p1.img_h = (int)img->h;
    p1.img_w = (int)img->w;
    p1.nq = nq;
    p1.nq_log = nq == 4 ? 2 : nq == 2 ? 1 : 0;
    p1.L = f.L;
    p1.scratch_img_rows = (int64_t)nq * f.Hp;
    const bool pitch16 = aligned16(img->data) && (img->row_stride * es) % 16 == 0 &&
                         (img->batch == 1 || (img->batch_stride * es) % 16 == 0);
#ifndef FHT_RANGE_TMA
#define FHT_RANGE_TMA 1
#endif
    // range: TMA rows + shared-memory gather when a tile row's source span fits one row load
    p1.fill_tma = pitch16 && (!rg || (FHT_RANGE_TMA && rg->alpha >= 1.0 && !rg->transposed));
    p1.fill_vec = f.m >= 2 && (es == 1 ? ((reinterpret_cast<uintptr_t>(img->data) & 3) == 0 &&
                                          img->row_stride % 4 == 0 && (img->batch == 1 || img->batch_stride % 4 == 0))
                                       : pitch16);
    // one TMA per image row (view [row][col/32][32]) for 4-byte images whose width is a multiple of 32
    p1.fill32 = FHT_ROW32 && p1.fill_tma && !rg && es == 4 && img->w % 32 == 0;
    int span1 = 1 << 30;
    for (int q = 0; q < nq; ++q) {
      v2::P1Slot& s = p1.slot[q];
      s.sigma = slots[q].sigma;
      s.transposed = slots[q].transposed;
      v2_pass1_range(f, s.sigma, rg, s.xlo, s.xhi, ses);
      s.srow0 = (int64_t)q * f.Hp;
      span1 = (s.xhi - s.xlo) < span1 ? (s.xhi - s.xlo) : span1;
    }
    p1.TX = span1 < v2::TX1 ? span1 : v2::TX1;
    if (sh) {  // each destination's box starts jper * TX elements into the staging plane: 128-byte aligned
      const int64_t jb = sh->J * ses;
      if ((jb * p1.TX) % 128 != 0) p1.TX = p1.TX >= 192 ? 192 : (p1.TX & ~31);
      if (p1.TX < 32 || (jb * p1.TX) % 128 != 0) return FHT_ERR_UNSUPPORTED;
    }
    int ntile1 = 0;
    for (int q = 0; q < nq; ++q) {
      v2::P1Slot& s = p1.slot[q];
      s.ntiles = (s.xhi - s.xlo + p1.TX - 1) / p1.TX;
      ntile1 = s.ntiles > ntile1 ? s.ntiles : ntile1;
    }
    if (rg) {
      p1.range = 1;
      p1.e_tab = rg->e_tab;
      p1.colmap = rg->colmap;
      p1.w_content = rg->w_content;
    }

    // pass-2 geometry
    v2::P2Params p2{};
    p2.scratch_img_rows = p1.scratch_img_rows;
    {
      const char* e = std::getenv("FHT_DEBUG_NO_TMA");
      p2.no_tma = (e && e[0] == '1') ? 1 : 0;
    }
    p2.nq = nq;
    p2.nq_log = p1.nq_log;
    p2.W = any ? (int)any->cols : f.W;
    p2.Hp = f.Hp;
    p2.wc = f.wc;
    const int span2 = rg ? rg->out_hi - rg->out_lo : p2.W;
    int box2 = v2::BOX2;
    if (box2 > (p2.W & ~3)) box2 = p2.W & ~3;
    if (box2 > (span2 & ~3)) box2 = span2 & ~3;
    p2.TX = box2 - v2::WO2;
    int ntile2 = 0;
    for (int q = 0; q < nq; ++q) {
      v2::P2Slot& s = p2.slot[q];
      s.sigma = slots[q].sigma;
      s.xlo1 = p1.slot[q].xlo;
      s.xhi1 = p1.slot[q].xhi;
      s.srow0 = p1.slot[q].srow0;
      if (rg) {
        s.xbeg = rg->out_lo;
        s.xend = rg->out_hi;
      } else {
        s.xbeg = s.sigma > 0 ? -(f.W - f.wc) : 0;  // signed columns [-pad, wc) (sigma = +1), [0, W)
        s.xend = s.xbeg + p2.W;
      }
      // sigma = +1 rows wrap at x = 0 (x < 0 is stored at x + W): no tile straddles it
      s.xmid = (!rg && s.sigma > 0 && s.xbeg < 0 && s.xend > 0) ? 0 : s.xbeg;
      auto part_tiles = [&](int lo, int hi) {
        if (hi <= lo) return 0;
        const int boxw = p2.TX + v2::WO2;
        return hi - lo <= boxw ? 1 : 1 + (hi - lo - boxw + p2.TX - 1) / p2.TX;
      };
      s.ntiles_a = part_tiles(s.xbeg, s.xmid);
      s.ntiles = s.ntiles_a + part_tiles(s.xmid, s.xend);
      ntile2 = s.ntiles > ntile2 ? s.ntiles : ntile2;
      s.qrow = slots[q].qrow;
      s.rbase = slots[q].row_base;
      s.rsign = slots[q].row_sign;
      s.skip = slots[q].skip_t;
    }
    p2.rows_out = 1 << 30;
    if (rg) {
      p2.range = 1;
      p2.start_tab = rg->start_tab;
      p2.len_tab = rg->len_tab;
      p2.rows_out = rg->rows;
    }
    P2Maps m2;
    CUtensorMap* tm_out[2] = {&m2.out0, &m2.out1};
    p2.ndest = 0;
    for (int d = 0; d < 2; ++d) {
      const fht_hough* o = outs.d[d];
      if (!o) continue;
      v2::P2Dest& D = p2.dest[p2.ndest];
      D.shifted = d;
      D.ptr = o->data;
      D.pitch = o->row_stride;
      D.rows_per_img = o->batch_stride / o->row_stride;
      D.nrows = o->batch * D.rows_per_img;
      if (!make_row_map(tm_out[p2.ndest], o->data, o->dtype == FHT_F32, (uint64_t)o->cols,
                        (uint64_t)(o->batch * D.rows_per_img), (uint64_t)o->row_stride, (uint32_t)box2))
        return FHT_ERR_CUDA;
      if (p2.ndest == 0 && !make_row_map(&m2.out0_box, o->data, o->dtype == FHT_F32, (uint64_t)o->cols,
                                         (uint64_t)(o->batch * D.rows_per_img), (uint64_t)o->row_stride,
                                         (uint32_t)box2, (uint32_t)v2::p2_box_rows(f.L)))
        return FHT_ERR_CUDA;
      ++p2.ndest;
    }
    if (p2.ndest == 1) m2.out1 = m2.out0;
    if (!outs.d[0]) m2.out0_box = m2.out0;
    const bool f32 = img->dtype == FHT_F32;
    if (sh) {
      const int64_t Z = img->batch * nq;
      const int logS = ilog2(sh->S);
      P1Maps m1s;
      P2Maps m2s = m2;
      if (sh->phase == 1) {  // pass 1 of strips [rank S, (rank + 1) S): every rank's groups to dst[h]
        p1.ndst = sh->world;
        p1.jper = (int)sh->J;
        p1.strip0 = (int)(sh->rank * sh->S);
        p1.L = logS;  // the grid's strips per image
        p1.z0 = 0;
        p1.img0 = 0;
        p1.ntiles = ntile1;
        for (int h = 0; h < sh->world; ++h)
          if (!make_dst_map(&m1s.dst.m[h], sh->dst[h], ses, f32, sp.pitch, sh->S, sh->J, Z, p1.TX, (int)sh->J))
            return FHT_ERR_CUDA;
        if (p1.fill_tma) {
          if (!make_p1_image_maps(&m1s.img0, &m1s.img1, img, p1, es)) return FHT_ERR_CUDA;
        } else {
          m1s.img0 = m1s.dst.m[0];
          m1s.img1 = m1s.dst.m[0];
        }
        if (!make_imgT_map(m1s, p1, img, f.m)) return FHT_ERR_CUDA;
        const dim3 g1((unsigned)(ntile1 * nq), (unsigned)sh->S, (unsigned)img->batch);
        log.before(st);
        cudaError_t e;
        switch (img->dtype) {
          case FHT_U8: e = launch_p1<uint8_t>(f.m, g1, m1s, p1, st); break;
          case FHT_I32: e = launch_p1<int32_t>(f.m, g1, m1s, p1, st); break;
          default: e = launch_p1<float>(f.m, g1, m1s, p1, st); break;
        }
        if (e != cudaSuccess) return FHT_ERR_CUDA;
        log.after(st);
        return 1;
      }
      // pass 2 of groups [rank J, (rank + 1) J) from the received chunks [g][z][j_local][strip_local]
      const uint64_t rows = (uint64_t)sh->world * sh->chunk_rows;
      p2.scr_rows = (int64_t)rows;
      void* recv = const_cast<void*>(sh->recv);
      if (!make_scr_maps(&m2s.scr0, &m2s.scr1, recv, f32, ses == 2, (uint64_t)span1, rows, (uint64_t)sp.pitch))
        return FHT_ERR_CUDA;
      p2.scratch_img_rows = nq * sh->J * sh->S;
      for (int q = 0; q < nq; ++q) p2.slot[q].srow0 = q * sh->J * sh->S;
      p2.row0 = 0;
      p2.img0 = 0;
      p2.j0 = (int)(sh->rank * sh->J);
      p2.logS = logS;
      p2.strideG = sh->chunk_rows;
      p2.ntiles = ntile2;
      p2.m = f.m;
      p2.ngroups = (int)sh->J;
      const dim3 g2((unsigned)ntile2, (unsigned)sh->J, (unsigned)(img->batch * nq));
      log.before(st);
      const cudaError_t e = f32 ? launch_p2<float>(f.L, g2, m2s, p2, st)
                                : ses == 2 ? launch_p2<int, uint16_t>(f.L, g2, m2s, p2, st)
                                           : launch_p2<int>(f.L, g2, m2s, p2, st);
      if (e != cudaSuccess) return FHT_ERR_CUDA;
      log.after(st);
      return 1;
    }
    const uint64_t scr_rows = pipe ? (uint64_t)pq.NBUF * pq.nbu * f.Hp : (uint64_t)sp.nbuf * sp.chunk * p1.scratch_img_rows;
    P1Maps m1;
    // pass-1 stores: scratch [z][j][strip][column], one box {TX, 1, ngroups, 1} per tile (shifts j < ngroups)
    p1.ndst = 1;
    p1.jper = ngroups;
    p1.strip0 = 0;
    p2.j0 = 0;
    p2.logS = f.L;
    p2.strideG = 0;
    p2.scr_rows = (int64_t)scr_rows;
    if (!make_dst_map(&m1.dst.m[0], ws, ses, f32, sp.pitch, nstrips, 1 << f.m, (int64_t)(scr_rows / f.Hp), p1.TX,
                      ngroups))
      return FHT_ERR_CUDA;
    if (p1.fill_tma) {
      if (!make_p1_image_maps(&m1.img0, &m1.img1, img, p1, es)) return FHT_ERR_CUDA;
    } else {
      m1.img0 = m1.dst.m[0];
      m1.img1 = m1.dst.m[0];
    }
    if (!make_imgT_map(m1, p1, img, f.m)) return FHT_ERR_CUDA;
    // persistent pass 1 (k_p1p): 64-row strips of 4-byte images with one-TMA rows, full-width tiles, all 64 shifts
    if (f.m == 6 && es == 4 && !rg && p1.fill_tma && p1.fill32 && p1.TX == v2::TX1 && ngroups == 64 && !pipe &&
        (int64_t)ntile1 * nq * nstrips * sp.chunk < (1ll << 30) && env_int("FHT_P1_PERSIST", 1) != 0) {
      if (!make_image_map32(&m1.img8, img, 8) || !make_image_map_swz(&m1.imgS, img) ||
          !make_dst_map(&m1.dst4, ws, ses, f32, sp.pitch, nstrips, 1 << f.m, (int64_t)(scr_rows / f.Hp), p1.TX,
                        v2::kP1pHalf))
        return FHT_ERR_CUDA;
      m1.persist = 1;
      m1.scr = ws;
      m1.scr_pitch = sp.pitch;
    } else if (f.m == 4 && es == 1 && ses == 2 && !rg && p1.fill_tma && p1.tfill_tma && img->w % 128 == 0 &&
               p1.TX == v2::TX1 && ngroups == 16 && !pipe && env_int("FHT_P1_PERSIST", 1) != 0 &&
               env_int("FHT_P1_PERSIST_U8", 1) != 0) {
      // 16-row strips of u8 images (k_p1p8): img8 = the [row][col/128][128] view, imgT = the transposed-tile map
      if (!make_image_map128(&m1.img8, img) ||
          !make_dst_map(&m1.dst4, ws, ses, f32, sp.pitch, nstrips, 1 << f.m, (int64_t)(scr_rows / f.Hp), p1.TX, 4))
        return FHT_ERR_CUDA;
      m1.persist = 1;
    } else if (f.m == 6 && es == 4 && rg && nq == 1 && p1.fill_tma && !p1.fill32 && p1.TX == v2::TX1 && !pipe &&
               env_int("FHT_P1_PERSIST", 1) != 0 && env_int("FHT_P1_PERSIST_RANGE", 1) != 0) {
      // the §4 range loader in the persistent kernel: the 256- and 36-column row maps stand in for img8 / imgS
      m1.img8 = m1.img0;
      m1.imgS = m1.img1;
      if (!make_dst_map(&m1.dst4, ws, ses, f32, sp.pitch, nstrips, 1 << f.m, (int64_t)(scr_rows / f.Hp), p1.TX,
                        v2::kP1pHalf))
        return FHT_ERR_CUDA;
      m1.persist = 1;
      m1.scr = ws;
      m1.scr_pitch = sp.pitch;
    }
    // scratch as pass 2 reads it: columns [0, span1) = what pass 1 wrote; TMA zero-fills the rest
    if (!make_scr_maps(&m2.scr0, &m2.scr1, ws, f32, ses == 2, (uint64_t)span1, scr_rows, (uint64_t)sp.pitch))
      return FHT_ERR_CUDA;

    if (pipe) {  // both passes in one persistent launch (fht_pipe.cuh)
      p1.ntiles = ntile1;
      p2.ntiles = ntile2;
      p2.m = f.m;
      p2.ngroups = ngroups;
      v2::PipeParams pp{};
      pp.nunits = pq.nunits;
      pp.nq = nq;
      pp.nbu = pq.nbu;
      pp.D = pq.D;
      pp.NBUF = pq.NBUF;
      pp.nstrips = nstrips;
      pp.ntiles1 = ntile1;
      pp.ngroups = ngroups;
      pp.ntiles2 = ntile2;
      pp.L = f.L;
      pp.buf_rows = (int64_t)pq.nbu * f.Hp;
      pp.counters = reinterpret_cast<int*>(static_cast<char*>(ws) + pq.scratch_bytes);
      if (const char* tp = std::getenv("FHT_PIPE_TRACE_PTR")) {  // debug hook: tools/pipe_trace.py
        pp.trace = reinterpret_cast<unsigned long long*>(std::strtoull(tp, nullptr, 0));
        pp.trace_n = env_int("FHT_PIPE_TRACE_N", 0);
      }
      PipeMaps pm{m1.img0, m1.img1, m1.dst, m2.scr0, m2.scr1, m2.out0, m2.out1, m2.out0_box};
      log.before(st);
      if (cudaMemsetAsync(pp.counters, 0, (size_t)(1 + 2 * pq.nunits) * sizeof(int), st) != cudaSuccess)
        return FHT_ERR_CUDA;
      if (launch_pipe(img->dtype == FHT_U8 ? 0 : img->dtype == FHT_I32 ? 1 : 2, f.m, f.L, pm, p1, p2, pp, st) !=
          cudaSuccess)
        return FHT_ERR_CUDA;
      log.after(st);
      return 1;
    }

    // Staggered pass pairs (fht_dual.cuh): chunks of dc images in two scratch buffers; launch k runs pass 1 of
    // chunk k beside pass 2 of chunk k - 1 in one grid. FHT_DUAL_IMGS = images per chunk (0: off).
    const int dual_imgs = env_int("FHT_DUAL_IMGS", 0);
    if (dual_imgs > 0 && !rg && dual_split_ok(f.m, f.L)) {
      const int64_t cap = sp.nbuf == 2 ? sp.chunk : sp.chunk / 2;  // images per buffer with two buffers
      const int64_t dc = dual_imgs < cap ? dual_imgs : cap;
      if (dc >= 1 && img->batch > dc) {
        const int nch = (int)((img->batch + dc - 1) / dc);
        const int dt = img->dtype == FHT_U8 ? 0 : img->dtype == FHT_I32 ? 1 : 2;
        const PipeMaps pm{m1.img0, m1.img1, m1.dst, m2.scr0, m2.scr1, m2.out0, m2.out1, m2.out0_box};
        p1.ntiles = ntile1;
        p2.ntiles = ntile2;
        p2.m = f.m;
        p2.ngroups = ngroups;
        auto set1 = [&](int k) {  // pass 1 of chunk k -> buffer k & 1
          p1.img0 = (int)(k * dc);
          p1.z0 = (int)((k & 1) * dc * nq);
          return (int)((img->batch - k * dc) < dc ? (img->batch - k * dc) : dc);
        };
        auto set2 = [&](int k) {
          p2.img0 = (int)(k * dc);
          p2.row0 = (k & 1) * dc * p1.scratch_img_rows;
          return (int)((img->batch - k * dc) < dc ? (img->batch - k * dc) : dc);
        };
        for (int k = 0; k <= nch; ++k) {
          cudaError_t e;
          log.before(st);
          if (k == 0) {
            const int nb = set1(0);
            const dim3 g1((unsigned)(ntile1 * nq), (unsigned)nstrips, (unsigned)nb);
            switch (img->dtype) {
              case FHT_U8: e = launch_p1<uint8_t>(f.m, g1, m1, p1, st); break;
              case FHT_I32: e = launch_p1<int32_t>(f.m, g1, m1, p1, st); break;
              default: e = launch_p1<float>(f.m, g1, m1, p1, st); break;
            }
          } else if (k == nch) {
            const int nb = set2(nch - 1);
            const dim3 g2((unsigned)ntile2, (unsigned)ngroups, (unsigned)(nb * nq));
            e = f32 ? launch_p2<float>(f.L, g2, m2, p2, st)
                    : ses == 2 ? launch_p2<int, uint16_t>(f.L, g2, m2, p2, st) : launch_p2<int>(f.L, g2, m2, p2, st);
          } else {
            const int nb1 = set1(k), nb2 = set2(k - 1);
            v2::DualParams dp{};
            dp.ntiles1 = ntile1;
            dp.nstrips = nstrips;
            dp.ntiles2 = ntile2;
            dp.ngroups = ngroups;
            dp.t1 = (int64_t)nb1 * nstrips * ntile1 * nq;
            dp.t2 = (int64_t)nb2 * nq * ngroups * ntile2;
            e = launch_dual(dt, f.m, f.L, pm, p1, p2, dp, st);
          }
          if (e != cudaSuccess) return FHT_ERR_CUDA;
          log.after(st);
          ++launches;
        }
        return launches;
      }
    }


    // Chunks of the batch; with an auxiliary stream and two scratch buffers, pass 1 of chunk k+1
    // (aux) overlaps pass 2 of chunk k (main): p2(k) waits for p1(k), p1(k+2) for p2(k).
    const int nchunks = (int)((img->batch + sp.chunk - 1) / sp.chunk);
    cudaStream_t aux = (log.opts && log.opts->aux_stream && sp.nbuf == 2 && nchunks > 1 &&
                        (cudaStream_t)log.opts->aux_stream != st)
                           ? (cudaStream_t)log.opts->aux_stream
                           : nullptr;
    cudaEvent_t ev_start = nullptr, ev_p1[2] = {nullptr, nullptr}, ev_p2[2] = {nullptr, nullptr};
    auto destroy_events = [&]() {
      for (cudaEvent_t e : {ev_start, ev_p1[0], ev_p1[1], ev_p2[0], ev_p2[1]})
        if (e) cudaEventDestroy(e);
    };
    if (aux) {
      bool ok = cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming) == cudaSuccess;
      for (int b = 0; b < 2; ++b) {
        ok = ok && cudaEventCreateWithFlags(&ev_p1[b], cudaEventDisableTiming) == cudaSuccess;
        ok = ok && cudaEventCreateWithFlags(&ev_p2[b], cudaEventDisableTiming) == cudaSuccess;
      }
      ok = ok && cudaEventRecord(ev_start, st) == cudaSuccess && cudaStreamWaitEvent(aux, ev_start, 0) == cudaSuccess;
      if (!ok) {
        destroy_events();
        return FHT_ERR_CUDA;
      }
    }
    const int64_t chunk_rows = (int64_t)sp.chunk * p1.scratch_img_rows;
    for (int k = 0; k < nchunks; ++k) {
      const int64_t b0 = (int64_t)k * sp.chunk;
      const int nb = (int)((img->batch - b0) < sp.chunk ? (img->batch - b0) : sp.chunk);
      const int buf = sp.nbuf == 2 ? (k & 1) : 0;
      p1.img0 = (int)b0;
      p2.img0 = (int)b0;
      p1.z0 = buf * sp.chunk * nq;
      p2.row0 = buf * chunk_rows;
      p1.ntiles = ntile1;
      dim3 g1((unsigned)(ntile1 * nq), (unsigned)nstrips, (unsigned)nb);
      cudaStream_t s1 = aux ? aux : st;
      if (aux && k >= 2 && cudaStreamWaitEvent(aux, ev_p2[buf], 0) != cudaSuccess) {
        destroy_events();
        return FHT_ERR_CUDA;
      }
      cudaError_t e;
      log.before(s1);
      switch (img->dtype) {
        case FHT_U8: e = launch_p1<uint8_t>(f.m, g1, m1, p1, s1); break;
        case FHT_I32: e = launch_p1<int32_t>(f.m, g1, m1, p1, s1); break;
        default: e = launch_p1<float>(f.m, g1, m1, p1, s1); break;
      }
      if (e != cudaSuccess) {
        destroy_events();
        return FHT_ERR_CUDA;
      }
      log.after(s1);
      ++launches;
      if (aux && (cudaEventRecord(ev_p1[buf], aux) != cudaSuccess || cudaStreamWaitEvent(st, ev_p1[buf], 0) != cudaSuccess)) {
        destroy_events();
        return FHT_ERR_CUDA;
      }
      p2.ntiles = ntile2;
      p2.m = f.m;
      p2.ngroups = ngroups;
      dim3 g2((unsigned)ntile2, (unsigned)ngroups, (unsigned)(nb * nq));
      e = f32 ? launch_p2<float>(f.L, g2, m2, p2, st)
              : ses == 2 ? launch_p2<int, uint16_t>(f.L, g2, m2, p2, st) : launch_p2<int>(f.L, g2, m2, p2, st);
      if (e != cudaSuccess) {
        destroy_events();
        return FHT_ERR_CUDA;
      }
      log.after(st);
      ++launches;
      if (aux && cudaEventRecord(ev_p2[buf], st) != cudaSuccess) {
        destroy_events();
        return FHT_ERR_CUDA;
      }
    }
    destroy_events();
    return launches;
  }

  // ---------------- v1 (degenerate frames only)
  const int Ws = (int)sp.pitch;
  const int nstrips = 1 << f.L, ngroups = 1 << f.m;
  for (int64_t b0 = 0; b0 < img->batch; b0 += sp.chunk) {
    const int nb = (int)((img->batch - b0) < sp.chunk ? (img->batch - b0) : sp.chunk);
    Pass1Args p1{};
    p1.img = img->data;
    p1.img_bstride = img->batch_stride;
    p1.img_rstride = img->row_stride;
    if (nq > 2) return FHT_ERR_UNSUPPORTED;  // v1 handles one orientation per launch
    p1.img_rows = f.rows_avail;
    p1.img_cols = f.cols_avail;
    p1.transposed = f.transposed;
    p1.scratch = ws;
    p1.scratch_zstride = (int64_t)f.Hp * Ws;
    p1.L = f.L;
    p1.Ws = Ws;
    p1.nq = nq;
    p1.img0 = (int)b0;
    for (int q = 0; q < nq; ++q) {
      p1.sigma[q] = slots[q].sigma;
      p1.xlo[q] = rg ? rg->x_lo : (slots[q].sigma > 0 ? -((1 << f.m) - 1) : 0);
    }
    if (rg) {
      p1.range = 1;
      p1.e_tab = rg->e_tab;
      p1.colmap = rg->colmap;
      p1.w_content = rg->w_content;
    }
    const int ntile1 = (Ws + kTileX - 1) / kTileX;
    dim3 g1(ntile1, nstrips, nb * nq);
    cudaError_t e;
    log.before(st);
    switch (img->dtype) {
      case FHT_U8: e = launch_pass1<uint8_t>(f.m, g1, p1, st); break;
      case FHT_I32: e = launch_pass1<int32_t>(f.m, g1, p1, st); break;
      default: e = launch_pass1<float>(f.m, g1, p1, st); break;
    }
    if (e != cudaSuccess) return FHT_ERR_CUDA;
    log.after(st);
    ++launches;

    for (int d = 0; d < 2; ++d) {
      const fht_hough* out = outs.d[d];
      if (!out) continue;
      Pass2Args p2{};
      p2.scratch = ws;
      p2.scratch_zstride = p1.scratch_zstride;
      p2.Ws = Ws;
      p2.m = f.m;
      p2.L = f.L;
      p2.out = out->data;
      p2.out_img_stride = out->batch_stride;
      p2.out_row_stride = out->row_stride;
      p2.W = (int)out->cols;
      p2.wc = f.wc;
      p2.Hp = f.Hp;
      p2.nq = nq;
      p2.img0 = (int)b0;
      p2.shift = d ? (rg ? 2 : 1) : 0;
      int span = p2.W;
      for (int q = 0; q < nq; ++q) {
        p2.sigma[q] = slots[q].sigma;
        p2.xlo[q] = p1.xlo[q];
        p2.out_q_offset[q] = slots[q].qrow * out->row_stride;
        p2.row_base[q] = slots[q].row_base;
        p2.row_sign[q] = slots[q].row_sign;
        p2.skip_t[q] = slots[q].skip_t;
        p2.xbeg[q] = rg ? rg->out_lo : (slots[q].sigma > 0 ? -f.Hp : 0);
      }
      if (rg) {
        p2.range = 1;
        p2.start_tab = rg->start_tab;
        p2.len_tab = rg->len_tab;
        span = rg->out_hi - rg->out_lo;
      }
      const int ntile2 = (span + kTileX - 1) / kTileX;
      dim3 g2(ntile2, ngroups, nb * nq);
      e = img->dtype == FHT_F32 ? launch_pass2<float>(f.L, g2, p2, st) : launch_pass2<int>(f.L, g2, p2, st);
      if (e != cudaSuccess) return FHT_ERR_CUDA;
      log.after(st);
      ++launches;
    }
  }
  return launches;
}

int validate_out(const fht_hough* out, const fht_hough& want) {
  if (!out->data) return FHT_ERR_ARG;
  if (out->dtype != want.dtype) return FHT_ERR_DTYPE;
  if (out->mode != want.mode || out->batch != want.batch || out->nquad != want.nquad ||
      out->rows != want.rows || out->cols != want.cols)
    return FHT_ERR_SHAPE;
  if (want.mode == FHT_MODE_FULL && out->layout != want.layout) return FHT_ERR_SHAPE;
  if (out->row_stride < out->cols) return FHT_ERR_SHAPE;
  // uniform row pitch across quadrants and images: the kernels address a [rows_total][W] view
  if (out->nquad > 1 && out->quad_stride != out->rows * out->row_stride) return FHT_ERR_SHAPE;
  const int64_t per_img = out->nquad * out->rows * out->row_stride;
  if (out->batch > 1 && (out->batch_stride < per_img || out->batch_stride % out->row_stride != 0))
    return FHT_ERR_SHAPE;
  if (out->batch == 1 && out->batch_stride % out->row_stride != 0) return FHT_ERR_SHAPE;
  if (!aligned16(out->data) || (out->row_stride & 3) != 0) return FHT_ERR_ALIGN;  // TMA row stores
  return FHT_OK;
}

bool overlaps(const void* a, size_t an, const void* b, size_t bn) {
  const char* pa = static_cast<const char*>(a);
  const char* pb = static_cast<const char*>(b);
  return pa < pb + bn && pb < pa + an;
}
size_t image_extent_bytes(const fht_image* img) {
  return ((size_t)(img->batch - 1) * img->batch_stride + (size_t)(img->h - 1) * img->row_stride + img->w) *
         dtype_size(img->dtype);
}
size_t hough_extent_bytes(const fht_hough* h) {
  const int64_t qs = h->nquad > 1 ? h->quad_stride : 0;
  return ((size_t)(h->batch - 1) * h->batch_stride + (size_t)(h->nquad - 1) * qs + (size_t)(h->rows - 1) * h->row_stride +
          h->cols) * 4;
}

// Validate the (out, out_shifted) pair against the wanted shape; no aliasing between any of
// image, outputs and workspace.
int validate_outs(const fht_image* img, const fht_hough* out, const fht_hough* out_s, const fht_hough& want,
                  const void* ws, size_t ws_bytes) {
  if (!out && !out_s) return FHT_ERR_ARG;
  if (ws && overlaps(ws, ws_bytes, img->data, image_extent_bytes(img))) return FHT_ERR_ARG;  // fht.h: no aliasing
  const fht_hough* o[2] = {out, out_s};
  for (int d = 0; d < 2; ++d) {
    if (!o[d]) continue;
    int s = validate_out(o[d], want);
    if (s) return s;
    if (overlaps(img->data, image_extent_bytes(img), o[d]->data, hough_extent_bytes(o[d]))) return FHT_ERR_ARG;
    if (ws && overlaps(ws, ws_bytes, o[d]->data, hough_extent_bytes(o[d]))) return FHT_ERR_ARG;
  }
  if (out && out_s && overlaps(out->data, hough_extent_bytes(out), out_s->data, hough_extent_bytes(out_s)))
    return FHT_ERR_ARG;
  return FHT_OK;
}

void mark_outs(fht_hough* out, fht_hough* out_s) {
  if (out) out->shifted = 0;
  if (out_s) out_s->shifted = 1;
}

// Plan geometry helpers (R13, R16, R17): identical double formulas to the device tables.
int plan_e(double g, int64_t y) {
  volatile double p = g * (double)y;  // volatile: forbid contraction into an FMA
  return (int)std::floor(p + 0.5);
}

// the plan's frame is the image, or its transpose for a mostly-horizontal plan
bool plan_matches(const fht_image* img, const fht_angle_plan_t* plan) {
  return plan->transposed ? (plan->h == img->w && plan->w == img->h) : (plan->h == img->h && plan->w == img->w);
}

Frame range_frame(const fht_image* img, const fht_angle_plan_t* plan) {
  Frame f{};
  f.transposed = plan->transposed ? 1 : 0;
  f.Hp = (int)plan->Hp;
  f.K = ilog2(f.Hp);
  f.wc = (int)plan->w_content;
  f.W = (int)plan->W;
  f.rows_avail = (int)plan->h;
  f.cols_avail = (int)plan->w;
  split_levels(f);
  return f;
}

RangeDev range_geometry(const Frame& f, const fht_angle_plan_t* plan) {
  RangeDev rg{};
  rg.w_content = (int)plan->w_content;
  rg.alpha = plan->alpha;
  rg.transposed = plan->transposed ? 1 : 0;
  rg.rows = (int)plan->rows;
  rg.x_lo = (int)plan->e_min - ((1 << f.m) - 1);
  rg.x_hi = (int)(plan->e_max + plan->w_content);
  // pass-2 signed columns: [min_s start_s, max_s start_s + W'); start_s >= e_min - (Hp-1) ...
  rg.out_lo = (int)plan->e_min - (f.Hp - 1);
  // ... and start_s = min_y (e_y - D_s(y)) <= e_min (D >= 0): no row stores at x >= e_min + W'
  rg.out_hi = (int)plan->e_min + (int)plan->W;
  return rg;
}

size_t range_tables_bytes(const fht_angle_plan_t* plan) {
  const size_t tables = (size_t)(plan->h + plan->w_content + 2 * plan->Hp + 64) * 4;
  return (tables + 255) & ~size_t(255);
}

}  // namespace

namespace {
// peaks: rows per band so that the band pass has about FHT_PEAKS_CTAS_PER_SM CTAs per SM (at most one band per plane height)
int peaks_band(const fht_hough* h) {
  const int64_t planes = h->batch * h->nquad;
#ifndef FHT_PEAKS_CTAS_PER_SM
#define FHT_PEAKS_CTAS_PER_SM 1  // measured: fewer, taller bands keep each warp's floor high (C3 0.35 -> 0.27 ms)
#endif
  constexpr int64_t kCtas = FHT_PEAKS_CTAS_PER_SM * 148;
  int64_t band = (h->rows * planes + kCtas - 1) / kCtas;
  if (band < 8) band = 8;
  if (band > h->rows) band = h->rows;
  return (int)band;
}
}  // namespace

extern "C" {

const char* fht_status_string(int s) {
  if (s >= 0) return "ok";
  switch (s) {
    case FHT_ERR_ARG: return "invalid argument";
    case FHT_ERR_DTYPE: return "unsupported dtype";
    case FHT_ERR_SHAPE: return "output shape mismatch";
    case FHT_ERR_ALIGN: return "pointer or pitch not 16-byte aligned";
    case FHT_ERR_UNSUPPORTED: return "unsupported on the GPU path";
    case FHT_ERR_WORKSPACE: return "workspace missing or too small";
    case FHT_ERR_STATE: return "descriptor already shifted";
    case FHT_ERR_CUDA: return "CUDA error";
  }
  return "unknown status";
}

namespace {
int plan_make(int64_t h, int64_t w, double tmin, double tmax, bool pruned, fht_angle_plan_t* out) {
  if (!out || h < 1 || w < 1) return FHT_ERR_ARG;
  if (!(tmin > -90.0 && tmin < tmax && tmax < 90.0)) return FHT_ERR_ARG;
  const double deg = M_PI / 180.0;
  const double k_lo = std::tan(tmin * deg), k_hi = std::tan(tmax * deg);
  const double alpha = pruned ? 1.0 : 1.0 / (k_hi - k_lo);
  if (!(alpha * (double)w >= 1.0)) return FHT_ERR_ARG;
  if (pruned && !(k_hi - k_lo <= 1.0)) return FHT_ERR_UNSUPPORTED;
  const int64_t Hp = next_pow2(h);
  if (Hp > 4096 || h > 4096) return FHT_ERR_UNSUPPORTED;
  const int64_t w_content = pruned ? w : (int64_t)std::ceil(alpha * (double)w - 1e-9);
  const double g = alpha * (-k_lo);
  // f2: rows s = (k - k_lo)(Hp - 1) for k in [k_lo, k_hi] (R19 in the sheared frame)
  int64_t rows = Hp;
  if (pruned) {
    const int64_t s_max = (int64_t)std::ceil((k_hi - k_lo) * (double)(Hp - 1) - 1e-9);
    rows = s_max + 1 < Hp ? s_max + 1 : Hp;
  }
  // e_y and the largest per-row spread of e_y - D_s(y) over y < h (R17). The min and max over y of
  // e_y - D_s(y) for every s come from the FHT's own block recursion with (min, max) in place of +
  // (D_t of a 2^k-row block = D_{t>>1} on its top half, ceil(t/2) + D_{t>>1} on its bottom half):
  //   mn_k[b][t] = min(mn_{k-1}[2b][t>>1], mn_{k-1}[2b+1][t>>1] - ceil(t/2))   (mx likewise),
  // Hp log2 Hp steps instead of Hp * h (a plan costs microseconds, so fht_angle_range can build it per call).
  int e_min = 1 << 30, e_max = -(1 << 30);
  constexpr int kInf = 1 << 29;  // neutral element (padding rows); |e_y|, D < 2^28 keep it apart
  int* buf = new int[4 * Hp];
  int *mn = buf, *mx = buf + Hp, *mn2 = buf + 2 * Hp, *mx2 = buf + 3 * Hp;
  for (int64_t y = 0; y < Hp; ++y) {
    if (y < h) {
      const int e = plan_e(g, y);
      e_min = e < e_min ? e : e_min;
      e_max = e > e_max ? e : e_max;
      mn[y] = mx[y] = e;
    } else {  // padding rows hold no pixel: neutral for min / max
      mn[y] = kInf;
      mx[y] = -kInf;
    }
  }
  for (int64_t half = 1; half < Hp; half <<= 1) {  // level: blocks of 2*half rows, shifts t < 2*half
    for (int64_t b = 0; b < Hp; b += 2 * half)
      for (int64_t t = 0; t < 2 * half; ++t) {
        const int64_t top = b + (t >> 1), bot = top + half;
        const int c = (int)((t + 1) >> 1);
        const int lo = mn[bot] - c, hi = mx[bot] - c;
        mn2[b + t] = mn[top] < lo ? mn[top] : lo;
        mx2[b + t] = mx[top] > hi ? mx[top] : hi;
      }
    std::swap(mn, mn2);
    std::swap(mx, mx2);
  }
  int64_t spread_max = 0;
  for (int64_t s = 0; s < rows; ++s)
    if ((int64_t)mx[s] - mn[s] > spread_max) spread_max = (int64_t)mx[s] - mn[s];
  delete[] buf;
  fht_angle_plan_t p{};
  p.theta_min_deg = tmin;
  p.theta_max_deg = tmax;
  p.k_lo = k_lo;
  p.k_hi = k_hi;
  p.alpha = alpha;
  p.g = g;
  p.h = h;
  p.w = w;
  p.Hp = Hp;
  p.w_content = w_content;
  p.W = w_content + (Hp > spread_max + 1 ? Hp : spread_max + 1);
  p.e_min = e_min;
  p.e_max = e_max;
  p.rows = rows;
  *out = p;
  return FHT_OK;
}
}  // namespace

int fht_angle_plan(int64_t h, int64_t w, double tmin, double tmax, fht_angle_plan_t* out) {
  return plan_make(h, w, tmin, tmax, false, out);
}

int fht_angle_of_row(const fht_angle_plan_t* plan, int64_t s, double* deg) {
  // R19 ("shift = h tg(phi)"): row s holds patterns of endpoint slope s / (Hp - 1) in the
  // transformed frame (D_s(Hp - 1) = s); undo the scale and the shear
  if (!plan || !deg || plan->Hp < 1 || s < 0 || s >= plan->Hp || !(plan->alpha > 0.0)) return FHT_ERR_ARG;
  const double k = plan->Hp > 1 ? plan->k_lo + (double)s / (plan->alpha * (double)(plan->Hp - 1)) : plan->k_lo;
  *deg = std::atan(k) * (180.0 / M_PI);
  return FHT_OK;
}

int fht_angle_plan_make_pruned(int64_t h, int64_t w, double tmin, double tmax, fht_angle_plan_t* out) {
  return plan_make(h, w, tmin, tmax, true, out);
}

int fht_angle_plan_make_ex(int64_t h, int64_t w, double tmin, double tmax, int32_t flags, fht_angle_plan_t* out) {
  if (flags & ~(FHT_PLAN_PRUNED | FHT_PLAN_HORIZONTAL)) return FHT_ERR_ARG;
  const bool hz = (flags & FHT_PLAN_HORIZONTAL) != 0;
  // mostly-horizontal: the vertical plan of the transposed image (frame h, w = image w, h)
  const int r = plan_make(hz ? w : h, hz ? h : w, tmin, tmax, (flags & FHT_PLAN_PRUNED) != 0, out);
  if (r == FHT_OK) out->transposed = hz ? 1 : 0;
  return r;
}

int fht_hough_describe(int mode, int layout, int quadrant, const fht_image* img, const fht_angle_plan_t* plan,
                       fht_hough* out) {
  if (!img || !out) return FHT_ERR_ARG;
  if (img->dtype != FHT_U8 && img->dtype != FHT_I32 && img->dtype != FHT_F32) return FHT_ERR_DTYPE;
  if (img->batch < 1 || img->h < 1 || img->w < 1) return FHT_ERR_ARG;
  fht_hough d{};
  d.dtype = out_dtype(img->dtype);
  d.mode = mode;
  d.layout = layout;
  d.batch = img->batch;
  d.h = img->h;
  d.w = img->w;
  d.Hp = next_pow2(img->h);
  d.Wp = next_pow2(img->w);
  d.quadrant = quadrant;
  if (mode == FHT_MODE_QUADRANT) {
    if (quadrant < 0 || quadrant > 3) return FHT_ERR_ARG;
    const bool tr = quadrant >= 2;
    d.nquad = 1;
    d.rows = tr ? d.Wp : d.Hp;
    d.cols = tr ? img->h + d.Wp : img->w + d.Hp;
  } else if (mode == FHT_MODE_FULL) {
    if (layout == FHT_LAYOUT_QUADS) {
      d.nquad = 4;
      d.rows = d.Hp > d.Wp ? d.Hp : d.Wp;
    } else if (layout == FHT_LAYOUT_CONCAT) {
      d.nquad = 1;
      d.rows = 2 * (d.Hp + d.Wp) - 3;
    } else {
      return FHT_ERR_ARG;
    }
    d.cols = d.Hp + d.Wp;
  } else if (mode == FHT_MODE_RANGE) {
    if (!plan || !plan_matches(img, plan)) return FHT_ERR_ARG;
    if (plan->rows < 1 || plan->rows > plan->Hp) return FHT_ERR_ARG;
    d.nquad = 1;
    d.rows = plan->rows;
    d.cols = plan->W;
    d.plan = *plan;
  } else {
    return FHT_ERR_ARG;
  }
  d.row_stride = (d.cols + 3) & ~int64_t(3);
  d.quad_stride = d.rows * d.row_stride;
  d.batch_stride = d.nquad * d.quad_stride;
  *out = d;
  return FHT_OK;
}

int fht_hough_describe_pad(int quadrant, const fht_image* img, int64_t pad_cols, fht_hough* out) {
  int s = fht_hough_describe(FHT_MODE_QUADRANT, 0, quadrant, img, nullptr, out);
  if (s || pad_cols == -1) return s;
  if (pad_cols < 0) return FHT_ERR_ARG;
  out->cols = (quadrant >= 2 ? img->h : img->w) + pad_cols;
  out->row_stride = (out->cols + 3) & ~int64_t(3);
  out->quad_stride = out->rows * out->row_stride;
  out->batch_stride = out->nquad * out->quad_stride;
  return FHT_OK;
}

size_t fht_quadrant_workspace_bytes(const fht_image* img, int quadrant, int64_t pad_cols) {
  const size_t base = fht_workspace_bytes(FHT_MODE_QUADRANT, img, nullptr);
  if (!img || pad_cols == -1 || quadrant < 0 || quadrant > 3) return base;
  const int64_t hf = quadrant >= 2 ? img->w : img->h;
  if (pad_cols >= hf - 1) return base;
  fht_hough d;
  if (fht_hough_describe(FHT_MODE_QUADRANT, 0, quadrant, img, nullptr, &d)) return 0;
  return (((size_t)(d.batch * d.batch_stride) * 4 + 255) & ~size_t(255)) + base;  // + the pad = Hp image
}

size_t fht_workspace_bytes(int mode, const fht_image* img, const fht_angle_plan_t* plan) {
  if (!img || img->batch < 1 || img->h < 1 || img->w < 1) return 0;
  if (mode == FHT_MODE_RANGE) {
    if (!plan) return 0;
    const Frame f = range_frame(img, plan);
    const RangeDev rg = range_geometry(f, plan);
    const ScratchPlan sp = scratch_plan(f, 1, 1, &rg, scratch_es(img->dtype));
    return ((sp.bytes + 255) & ~size_t(255)) + range_tables_bytes(plan);
  }
  size_t need = 0;
  const int es = scratch_es(img->dtype);
  if (mode == FHT_MODE_FULL && next_pow2(img->h) == next_pow2(img->w)) {
    const Frame f = make_frame(img->h, img->w, 0, 1);
    if (use_v2(f, nullptr)) {  // one 4-slot pass (two-launch schedule or the pipelined kernel)
      const size_t a = scratch_plan(f, 4, img->batch, nullptr, es).bytes, b = pipe_plan(f, 4, img->batch, nullptr, es).bytes;
      return a > b ? a : b;
    }
  }
  for (int tr = 0; tr < 2; ++tr) {
    const Frame f = make_frame(img->h, img->w, tr, mode == FHT_MODE_FULL);
    const int nq = mode == FHT_MODE_FULL ? 2 : 1;
    const size_t a = scratch_plan(f, nq, img->batch, nullptr, es).bytes, b = pipe_plan(f, nq, img->batch, nullptr, es).bytes;
    need = a > need ? a : need;
    need = b > need ? b : need;
  }
  return need;
}

}  // extern "C"

namespace {
// fht_quadrant with the caller's launch log (events / counts shared with the fold path's inner call)
int quadrant_run(const fht_image* img, int quadrant, int64_t pad_cols, fht_hough* out, fht_hough* out_shifted,
                 void* ws, size_t ws_bytes, fht_stream_t stream, LaunchLog& log) {
  int s = check_image(img);
  if (s) return s;
  if (quadrant < 0 || quadrant > 3) return FHT_ERR_ARG;
  // pad (R22): any pad >= h_frame - 1 keeps every line's signed columns apart mod
  // w + pad (rows >= h are zero, so no pattern reaches further than h - 1 columns); a smaller
  // pad folds lines cyclically: computed as the default transform + a fold
  const int64_t hf = quadrant >= 2 ? img->w : img->h;
  if (pad_cols < -1) return FHT_ERR_ARG;
  fht_hough want;
  s = fht_hough_describe_pad(quadrant, img, pad_cols, &want);
  if (s) return s;
  if (pad_cols != -1 && pad_cols < hf - 1) {
    // lines fold cyclically mod w + pad: the default (pad = Hp) transform into the workspace, then
    // the fold (k_fold; R22). Workspace: [temporary Hough image][scratch]
    if ((s = validate_outs(img, out, out_shifted, want, ws, ws_bytes))) return s;
    if ((out && out->quadrant != quadrant) || (out_shifted && out_shifted->quadrant != quadrant)) return FHT_ERR_ARG;
    fht_hough tmpd;
    if ((s = fht_hough_describe(FHT_MODE_QUADRANT, 0, quadrant, img, nullptr, &tmpd))) return s;
    const size_t tmp_bytes = ((size_t)(tmpd.batch * tmpd.batch_stride) * 4 + 255) & ~size_t(255);
    const size_t need = fht_quadrant_workspace_bytes(img, quadrant, pad_cols);
    if (!ws || ws_bytes < need) return FHT_ERR_WORKSPACE;
    tmpd.data = ws;
    const int r = quadrant_run(img, quadrant, -1, &tmpd, nullptr, static_cast<char*>(ws) + tmp_bytes,
                               ws_bytes - tmp_bytes, stream, log);
    if (r < 0) return r;
    FoldArgs fa{};
    fa.tmp = ws;
    fa.tmp_pitch = tmpd.row_stride;
    fa.tmp_batch = tmpd.batch_stride;
    if (out) {
      fa.out = out->data;
      fa.out_pitch = out->row_stride;
      fa.out_batch = out->batch_stride;
    }
    if (out_shifted) {
      fa.outs = out_shifted->data;
      fa.outs_pitch = out_shifted->row_stride;
      fa.outs_batch = out_shifted->batch_stride;
    }
    fa.Hp = (int)tmpd.rows;
    fa.W = (int)want.cols;
    fa.Wt = (int)tmpd.cols;
    fa.sigma = (quadrant == FHT_QA || quadrant == FHT_QD) ? 1 : -1;
    fa.pad = (int)(want.cols - (quadrant >= 2 ? img->h : img->w));  // fused fhtshift: R11 rule of this pad
    fa.xlo = fa.sigma > 0 ? -fa.Hp : 0;  // the default run's tiling window [xlo, xlo + Wt)
    fa.total = tmpd.batch * (int64_t)fa.Hp * fa.W;
    const int64_t nblk = std::min<int64_t>((fa.total + kThreads - 1) / kThreads, 148 * 16);
    // the inner run's last log.after() recorded the event that opens this launch
    if (tmpd.dtype == FHT_F32) k_fold<float><<<(unsigned)nblk, kThreads, 0, (cudaStream_t)stream>>>(fa);
    else k_fold<int><<<(unsigned)nblk, kThreads, 0, (cudaStream_t)stream>>>(fa);
    if (cudaGetLastError() != cudaSuccess) return FHT_ERR_CUDA;
    log.after((cudaStream_t)stream);
    mark_outs(out, out_shifted);
    return r + 1;
  }
  const Frame f = make_frame(img->h, img->w, quadrant >= 2, 0, pad_cols);
  if (pad_cols != -1 && pad_cols != f.Hp && !use_v2(f, nullptr)) return FHT_ERR_UNSUPPORTED;
  if ((s = validate_outs(img, out, out_shifted, want, ws, ws_bytes))) return s;
  if ((out && out->quadrant != quadrant) || (out_shifted && out_shifted->quadrant != quadrant)) return FHT_ERR_ARG;
  if ((s = check_frame_supported(f))) return s;
  Slot sl{};
  sl.sigma = (quadrant == FHT_QA || quadrant == FHT_QD) ? 1 : -1;
  sl.transposed = f.transposed;
  sl.qrow = 0;
  sl.row_base = 0;
  sl.row_sign = 1;
  sl.skip_t = -1;
  Outs o{{out, out_shifted}};
  const int r = run_orientation(img, f, &sl, 1, o, ws, ws_bytes, (cudaStream_t)stream, nullptr, log);
  if (r > 0) mark_outs(out, out_shifted);
  return r;
}
}  // namespace

extern "C" {

int fht_quadrant(const fht_image* img, int quadrant, int64_t pad_cols, fht_hough* out, fht_hough* out_shifted,
                 void* ws, size_t ws_bytes, fht_stream_t stream, const fht_exec_opts* opts) {
  LaunchLog log{opts, 0};
  return quadrant_run(img, quadrant, pad_cols, out, out_shifted, ws, ws_bytes, stream, log);
}

}  // extern "C"

namespace {
// sharded transform: validate (img, sh) against a fresh description
int shard_check(const fht_image* img, const fht_shard* sh) {
  if (!sh) return FHT_ERR_ARG;
  fht_shard want;
  const int s = fht_shard_describe(img, sh->world, sh->rank, &want);
  if (s) return s;
  if (want.chunk_bytes != sh->chunk_bytes || want.pitch != sh->pitch || want.S != sh->S || want.J != sh->J)
    return FHT_ERR_ARG;
  return FHT_OK;
}
void quads_slots(Slot* sl, int64_t rows_per_quad, int64_t row_base) {
  const int qid[4] = {FHT_QA, FHT_QB, FHT_QC, FHT_QD};
  for (int k = 0; k < 4; ++k) {
    sl[k].sigma = (qid[k] == FHT_QA || qid[k] == FHT_QD) ? 1 : -1;
    sl[k].transposed = qid[k] >= FHT_QC;
    sl[k].qrow = (int64_t)qid[k] * rows_per_quad;
    sl[k].row_base = (int)row_base;
    sl[k].row_sign = 1;
    sl[k].skip_t = -1;
  }
}
}  // namespace

extern "C" {

int fht_shard_describe(const fht_image* img, int world, int rank, fht_shard* out) {
  if (!img || !out) return FHT_ERR_ARG;
  if (img->dtype != FHT_U8 && img->dtype != FHT_I32 && img->dtype != FHT_F32) return FHT_ERR_DTYPE;
  if (img->batch < 1 || img->h < 1 || img->w < 1) return FHT_ERR_ARG;
  if (world < 1 || (world & (world - 1)) || rank < 0 || rank >= world) return FHT_ERR_ARG;
  if (world > v2::kMaxDst) return FHT_ERR_UNSUPPORTED;
  if (next_pow2(img->h) != next_pow2(img->w)) return FHT_ERR_UNSUPPORTED;  // one frame for all four slots
  const Frame f = make_frame(img->h, img->w, 0, 1);
  if (check_frame_supported(f) || !use_v2(f, nullptr)) return FHT_ERR_UNSUPPORTED;
  if ((1 << f.m) % world || (1 << f.L) % world) return FHT_ERR_UNSUPPORTED;
  fht_shard d{};
  d.world = world;
  d.rank = rank;
  d.m = f.m;
  d.L = f.L;
  d.S = (1 << f.L) / world;
  d.J = (1 << f.m) / world;
  d.rows_per_rank = f.Hp / world;
  d.scratch_es = scratch_es(img->dtype);
  d.pitch = v2_scratch_pitch(f, nullptr, d.scratch_es);
  d.chunk_rows = img->batch * 4 * d.J * d.S;
  d.chunk_bytes = d.chunk_rows * d.pitch * d.scratch_es;
  d.send_bytes = d.recv_bytes = world * d.chunk_bytes;
  int s = fht_hough_describe(FHT_MODE_FULL, FHT_LAYOUT_QUADS, 0, img, nullptr, &d.band);
  if (s) return s;
  d.band.rows = d.rows_per_rank;
  d.band.row0 = rank * d.rows_per_rank;
  d.band.quad_stride = d.band.rows * d.band.row_stride;
  d.band.batch_stride = d.band.nquad * d.band.quad_stride;
  *out = d;
  return FHT_OK;
}

int fht_shard_pass1(const fht_image* img, const fht_shard* sh, void* const* dst, fht_stream_t stream) {
  int s = check_image(img);
  if (s) return s;
  if ((s = shard_check(img, sh))) return s;
  if (!dst) return FHT_ERR_ARG;
  for (int h = 0; h < sh->world; ++h)
    if (!dst[h] || !aligned16(dst[h])) return dst[h] ? FHT_ERR_ALIGN : FHT_ERR_ARG;
  const Frame f = make_frame(img->h, img->w, 0, 1);
  Slot sl[4];
  quads_slots(sl, sh->rows_per_rank, -sh->band.row0);
  ShardCfg cfg{sh->world, sh->rank, 1, sh->S, sh->J, dst, nullptr, sh->chunk_rows};
  Outs o{{nullptr, nullptr}};
  LaunchLog log{nullptr, 0};
  return run_orientation(img, f, sl, 4, o, nullptr, 0, (cudaStream_t)stream, nullptr, log, &cfg);
}

int fht_shard_pass2(const fht_image* img, const fht_shard* sh, const void* recv, fht_hough* band,
                    fht_hough* band_shifted, fht_stream_t stream) {
  int s = check_image(img);
  if (s) return s;
  if ((s = shard_check(img, sh))) return s;
  if (!recv || (!band && !band_shifted)) return FHT_ERR_ARG;
  if (!aligned16(recv)) return FHT_ERR_ALIGN;
  for (fht_hough* o : {band, band_shifted}) {
    if (!o) continue;
    if ((s = validate_out(o, sh->band))) return s;
    if (o->row0 != sh->band.row0) return FHT_ERR_SHAPE;
    if (overlaps(recv, (size_t)sh->recv_bytes, o->data, hough_extent_bytes(o))) return FHT_ERR_ARG;
  }
  if (band && band_shifted && overlaps(band->data, hough_extent_bytes(band), band_shifted->data,
                                       hough_extent_bytes(band_shifted)))
    return FHT_ERR_ARG;
  const Frame f = make_frame(img->h, img->w, 0, 1);
  Slot sl[4];
  quads_slots(sl, sh->rows_per_rank, -sh->band.row0);
  ShardCfg cfg{sh->world, sh->rank, 2, sh->S, sh->J, nullptr, recv, sh->chunk_rows};
  Outs o{{band, band_shifted}};
  LaunchLog log{nullptr, 0};
  const int r = run_orientation(img, f, sl, 4, o, nullptr, 0, (cudaStream_t)stream, nullptr, log, &cfg);
  if (r > 0) mark_outs(band, band_shifted);
  return r;
}

int fht_full(const fht_image* img, int layout, fht_hough* out, fht_hough* out_shifted, void* ws, size_t ws_bytes,
             fht_stream_t stream, const fht_exec_opts* opts) {
  int s = check_image(img);
  if (s) return s;
  fht_hough want;
  if ((s = fht_hough_describe(FHT_MODE_FULL, layout, 0, img, nullptr, &want))) return s;
  if ((s = validate_outs(img, out, out_shifted, want, ws, ws_bytes))) return s;
  const int Hp = (int)want.Hp, Wp = (int)want.Wp;
  Outs o{{out, out_shifted}};
  LaunchLog log{opts, 0};
  Slot sl[4];
  // orientation 0: QA (+), QB (-); orientation 1: QC (-), QD (+)   (R4)
  const int qid[4] = {FHT_QA, FHT_QB, FHT_QC, FHT_QD};
  for (int k = 0; k < 4; ++k) {
    const int q = qid[k];
    sl[k].sigma = (q == FHT_QA || q == FHT_QD) ? 1 : -1;
    sl[k].transposed = q >= FHT_QC;
    if (layout == FHT_LAYOUT_QUADS) {
      sl[k].qrow = (int64_t)q * want.rows;
      sl[k].row_base = 0;
      sl[k].row_sign = 1;
      sl[k].skip_t = -1;
    } else {  // CONCAT (R7, R8)
      sl[k].qrow = 0;
      switch (q) {
        case FHT_QA: sl[k].row_base = Hp - 1; sl[k].row_sign = -1; sl[k].skip_t = -1; break;
        case FHT_QB: sl[k].row_base = Hp - 1; sl[k].row_sign = 1; sl[k].skip_t = 0; break;
        case FHT_QC: sl[k].row_base = 2 * Hp - 2 + Wp - 1; sl[k].row_sign = -1; sl[k].skip_t = Wp - 1; break;
        default: sl[k].row_base = 2 * Hp + Wp - 3; sl[k].row_sign = 1; sl[k].skip_t = 0; break;
      }
    }
  }
  const Frame f0 = make_frame(img->h, img->w, 0, 1), f1 = make_frame(img->h, img->w, 1, 1);
  if ((s = check_frame_supported(f0)) || (s = check_frame_supported(f1))) return s;
  int r;
#ifndef FHT_SPLIT_ORIENT
#define FHT_SPLIT_ORIENT 1
#endif
  // Square, one chunk, an auxiliary stream and no per-kernel events: QA/QB on `stream` and QC/QD
  // on the auxiliary stream, each a (pass 1, pass 2) pair over its own half of the 4-slot scratch,
  // so the latency-bound pass 1 of one orientation overlaps the store-bound pass 2 of the other.
  cudaStream_t aux = (opts && opts->aux_stream && (cudaStream_t)opts->aux_stream != (cudaStream_t)stream &&
                      !(opts->events && opts->n_events > 0))
                         ? (cudaStream_t)opts->aux_stream
                         : nullptr;
  const ScratchPlan sp2 = scratch_plan(f0, 2, img->batch, nullptr, scratch_es(img->dtype));
  const size_t half = (sp2.bytes + 255) & ~size_t(255);
  const bool pipe4 = Hp == Wp && pipe_plan(f0, 4, img->batch, nullptr, scratch_es(img->dtype)).on;
  // one image only: for a batch the merged 4-slot launches measured faster (C5 1.386 vs 1.414 ms,
  // profiles/r02/split_ab.log)
  if (FHT_SPLIT_ORIENT && aux && !pipe4 && (img->batch == 1 || env_int("FHT_SPLIT_BATCH", 0)) && Hp == Wp && use_v2(f0, nullptr) && sp2.nbuf == 1 &&
      sp2.chunk >= img->batch && 2 * half <= ws_bytes) {
    cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
    auto destroy = [&]() {
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
    };
    // FHT_SPLIT_STAGGER=1: the auxiliary orientation starts when the main one's pass 1 has completed, so
    // its pass 1 runs beside the main pass 2 instead of beside the main pass 1
    const bool stagger = env_int("FHT_SPLIT_STAGGER", 0) != 0;
    if (cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[2], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev[0], (cudaStream_t)stream) != cudaSuccess) {
      destroy();
      return FHT_ERR_CUDA;
    }
    LaunchLog quiet{nullptr, 0}, first{nullptr, 0, stagger ? ev[2] : nullptr};
    r = run_orientation(img, f0, sl, 2, o, ws, half, (cudaStream_t)stream, nullptr, first);
    if (cudaStreamWaitEvent(aux, stagger ? ev[2] : ev[0], 0) != cudaSuccess) {
      destroy();
      return FHT_ERR_CUDA;
    }
    const int r2 = r < 0 ? r : run_orientation(img, f0, sl + 2, 2, o, static_cast<char*>(ws) + half, half, aux, nullptr,
                                               quiet);
    const bool ok = cudaEventRecord(ev[1], aux) == cudaSuccess &&
                    cudaStreamWaitEvent((cudaStream_t)stream, ev[1], 0) == cudaSuccess;
    destroy();
    if (r < 0) return r;
    if (r2 < 0) return r2;
    if (!ok) return FHT_ERR_CUDA;
    r += r2;
  } else if (Hp == Wp && use_v2(f0, nullptr)) {
    // square: both orientations share one frame -> one pass-1 and one pass-2 launch for all four
    r = run_orientation(img, f0, sl, 4, o, ws, ws_bytes, (cudaStream_t)stream, nullptr, log);
    if (r < 0) return r;
  } else {
    r = run_orientation(img, f0, sl, 2, o, ws, ws_bytes, (cudaStream_t)stream, nullptr, log);
    if (r < 0) return r;
    const int r2 = run_orientation(img, f1, sl + 2, 2, o, ws, ws_bytes, (cudaStream_t)stream, nullptr, log);
    if (r2 < 0) return r2;
    r += r2;
  }
  mark_outs(out, out_shifted);
  return r;
}

size_t fht_angle_range_workspace_bytes(const fht_image* img, double theta_min_deg, double theta_max_deg) {
  fht_angle_plan_t p;
  if (!img || fht_angle_plan(img->h, img->w, theta_min_deg, theta_max_deg, &p) != FHT_OK) return 0;
  return fht_workspace_bytes(FHT_MODE_RANGE, img, &p);
}

int fht_angle_range(const fht_image* img, double theta_min_deg, double theta_max_deg, fht_hough* out,
                    fht_hough* out_shifted, void* ws, size_t ws_bytes, fht_stream_t stream, const fht_exec_opts* opts) {
  // P:117 "perform a transform for an arbitrary range of angles [gamma1; gamma2]": the §4 plan is
  // built here (host, O(Hp log Hp)) and must describe the same transform as the outputs
  int s = check_image(img);
  if (s) return s;
  fht_angle_plan_t p;
  if ((s = fht_angle_plan(img->h, img->w, theta_min_deg, theta_max_deg, &p))) return s;
  for (const fht_hough* o : {(const fht_hough*)out, (const fht_hough*)out_shifted}) {
    if (!o) continue;
    if (o->mode != FHT_MODE_RANGE || o->plan.transposed || o->plan.rows != p.rows || o->plan.W != p.W ||
        o->plan.w_content != p.w_content || o->plan.theta_min_deg != theta_min_deg ||
        o->plan.theta_max_deg != theta_max_deg)
      return FHT_ERR_SHAPE;
  }
  return fht_angle_range_plan(img, &p, out, out_shifted, ws, ws_bytes, stream, opts);
}

int fht_angle_range_plan(const fht_image* img, const fht_angle_plan_t* plan, fht_hough* out, fht_hough* out_shifted,
                         void* ws, size_t ws_bytes, fht_stream_t stream, const fht_exec_opts* opts) {
  int s = check_image(img);
  if (s) return s;
  if (!plan || !plan_matches(img, plan)) return FHT_ERR_ARG;
  fht_hough want;
  if ((s = fht_hough_describe(FHT_MODE_RANGE, 0, 0, img, plan, &want))) return s;
  if ((s = validate_outs(img, out, out_shifted, want, ws, ws_bytes))) return s;
  const size_t need = fht_workspace_bytes(FHT_MODE_RANGE, img, plan);
  if (!ws || ws_bytes < need) return FHT_ERR_WORKSPACE;
  const Frame f = range_frame(img, plan);
  if ((s = check_frame_supported(f))) return s;
  RangeDev rg = range_geometry(f, plan);
  const ScratchPlan sp = scratch_plan(f, 1, 1, &rg, scratch_es(img->dtype));
  if (plan->rows < f.Hp && !sp.v2) return FHT_ERR_UNSUPPORTED;  // pruned plans: v2 kernels only
  // workspace: [scratch][e_tab h][colmap w'][start Hp][len Hp]
  const size_t scratch = (sp.bytes + 255) & ~size_t(255);
  int* tab = reinterpret_cast<int*>(static_cast<char*>(ws) + scratch);
  rg.e_tab = tab;  // frame rows (image columns for a transposed plan)
  rg.colmap = tab + plan->h;
  rg.start_tab = tab + plan->h + plan->w_content;
  rg.len_tab = rg.start_tab + f.Hp;
  RangeTableArgs ta{};
  ta.g = plan->g;
  ta.alpha = plan->alpha;
  ta.h = (int)plan->h;  // the frame's rows / columns
  ta.w = (int)plan->w;
  ta.w_content = (int)plan->w_content;
  ta.Hp = f.Hp;
  ta.K = f.K;
  ta.e_tab = const_cast<int*>(rg.e_tab);
  ta.colmap = const_cast<int*>(rg.colmap);
  ta.start_tab = const_cast<int*>(rg.start_tab);
  ta.len_tab = const_cast<int*>(rg.len_tab);
  const int nb_tab = (f.Hp + kRangeRowsPerBlock - 1) / kRangeRowsPerBlock +
                     (int)((std::max<int64_t>(plan->h, plan->w_content) + kThreads - 1) / kThreads);
  LaunchLog log{opts, 0};
  log.before((cudaStream_t)stream);
  if (env_int("FHT_RANGE_TABLES_REC", 1) != 0) {  // supports by the (min, max) block recursion in one block
    const size_t smem = 4 * (size_t)f.Hp * sizeof(int);
    static std::atomic<unsigned long long> done{0};
    if (smem_optin(k_range_tables_rec, 4 * (size_t)4096 * sizeof(int), done) != cudaSuccess) return FHT_ERR_CUDA;
    const int nb = 1 + (int)((std::max<int64_t>(plan->h, plan->w_content) + kRangeRecThreads - 1) / kRangeRecThreads);
    k_range_tables_rec<<<nb, kRangeRecThreads, smem, (cudaStream_t)stream>>>(ta);
  } else {
    k_range_tables<<<nb_tab, kThreads, (size_t)plan->h * sizeof(int), (cudaStream_t)stream>>>(ta);
  }
  if (cudaGetLastError() != cudaSuccess) return FHT_ERR_CUDA;
  log.after((cudaStream_t)stream);
  Slot sl{};
  sl.sigma = 1;
  sl.transposed = plan->transposed ? 1 : 0;  // mostly-horizontal: the loader reads I[colmap[u]][y]
  sl.row_sign = 1;
  sl.skip_t = -1;
  Outs o{{out, out_shifted}};
  const int r = run_orientation(img, f, &sl, 1, o, ws, scratch, (cudaStream_t)stream, &rg, log);
  if (r < 0) return r;
  mark_outs(out, out_shifted);
  return r + 1;
}

int fhtshift(const fht_hough* in, fht_hough* out, fht_stream_t stream) {
  if (!in || !out || !in->data || !out->data) return FHT_ERR_ARG;
  if (in->shifted) return FHT_ERR_STATE;
  if (in->dtype != out->dtype || (in->dtype != FHT_I32 && in->dtype != FHT_F32)) return FHT_ERR_DTYPE;
  if (in->mode != out->mode || in->layout != out->layout || in->batch != out->batch || in->nquad != out->nquad ||
      in->rows != out->rows || in->cols != out->cols || in->Hp != out->Hp || in->Wp != out->Wp ||
      in->quadrant != out->quadrant)
    return FHT_ERR_SHAPE;
  if (overlaps(in->data, hough_extent_bytes(in), out->data, hough_extent_bytes(out))) return FHT_ERR_ARG;
  if (in->rows < 1 || in->cols < 1 || in->batch < 1) return FHT_ERR_ARG;
  ShiftArgs a{};
  a.in = in->data;
  a.out = out->data;
  a.in_img_stride = in->batch_stride;
  a.in_q_stride = in->quad_stride;
  a.in_row_stride = in->row_stride;
  a.out_img_stride = out->batch_stride;
  a.out_q_stride = out->quad_stride;
  a.out_row_stride = out->row_stride;
  a.rows = (int)in->rows;
  a.row0 = (int)in->row0;  // a shard's band: row r is shift row0 + r
  if (in->row0 != out->row0 || (in->row0 && in->mode != FHT_MODE_FULL)) return FHT_ERR_SHAPE;
  a.W = (int)in->cols;
  a.nquad = (int)in->nquad;
  a.rows_total = in->batch * in->nquad * in->rows;
  a.mode = in->mode;
  a.layout = in->layout;
  a.quadrant = in->quadrant;
  a.vec = a.W % 4 == 0 && aligned16(in->data) && aligned16(out->data);
  for (int64_t st : {in->batch_stride, in->quad_stride, in->row_stride, out->batch_stride, out->quad_stride,
                     out->row_stride})
    a.vec = a.vec && st % 4 == 0;
  size_t smem = 0;
  if (in->mode == FHT_MODE_QUADRANT) {
    a.Hp = a.Wp = (int)in->rows;  // the quadrant's own row count
    a.pad = (int)(in->cols - (in->quadrant >= 2 ? in->h : in->w));  // W - w_frame (R11 generic rule)
  } else if (in->mode == FHT_MODE_FULL) {
    a.Hp = (int)in->Hp;
    a.Wp = (int)in->Wp;
  } else {
    a.g = in->plan.g;
    a.h = (int)in->plan.h;
    a.K = ilog2(in->plan.Hp);
    a.w_content = (int)in->plan.w_content;
    smem = (size_t)a.h * sizeof(int);  // e_y table of the block (h <= 4096)
  }
  const int64_t nblk = (a.rows_total + kThreads / 32 - 1) / (kThreads / 32);
  if (in->dtype == FHT_F32) k_fhtshift<float><<<(unsigned)nblk, kThreads, smem, (cudaStream_t)stream>>>(a);
  else k_fhtshift<int><<<(unsigned)nblk, kThreads, smem, (cudaStream_t)stream>>>(a);
  if (cudaGetLastError() != cudaSuccess) return FHT_ERR_CUDA;
  out->shifted = 1;
  return 1;
}

size_t fht_peaks_workspace_bytes(const fht_hough* h) {
  if (!h || h->batch < 1 || h->nquad < 1 || h->rows < 1 || h->cols < 1) return 0;
  const int band = peaks_band(h);
  const int64_t nbands = (h->rows + band - 1) / band;
  // [planes][nbands][32] list keys, then [planes] thresholds
  return (size_t)(h->batch * h->nquad * nbands) * pk::kMaxK * sizeof(uint64_t) +
         (size_t)(h->batch * h->nquad) * sizeof(uint64_t);
}

int fht_peaks(const fht_hough* h, int32_t k, void* values, int32_t* rows, int32_t* cols, void* ws, size_t ws_bytes,
              fht_stream_t stream) {
  if (!h || !h->data || !values || !rows || !cols) return FHT_ERR_ARG;
  if (h->dtype != FHT_I32 && h->dtype != FHT_F32) return FHT_ERR_DTYPE;
  if (k < 1 || k > pk::kMaxK || h->batch < 1 || h->nquad < 1 || h->rows < 1 || h->cols < 1) return FHT_ERR_ARG;
  if (h->rows * h->cols >= (int64_t(1) << 32) - 1 || h->rows >= (int64_t(1) << 31)) return FHT_ERR_UNSUPPORTED;
  if (h->batch * h->nquad > 65535) return FHT_ERR_UNSUPPORTED;  // planes are gridDim.y of the band pass
  const size_t need = fht_peaks_workspace_bytes(h);
  if (!ws || ws_bytes < need) return FHT_ERR_WORKSPACE;
  pk::PeakArgs a{};
  a.data = h->data;
  a.bstride = h->batch_stride;
  a.qstride = h->quad_stride;
  a.rstride = h->row_stride;
  a.nquad = (int)h->nquad;
  a.R = (int)h->rows;
  a.W = (int)h->cols;
  a.band = peaks_band(h);
  a.nbands = (a.R + a.band - 1) / a.band;
  a.part = static_cast<uint64_t*>(ws);
  a.thr = reinterpret_cast<unsigned long long*>(a.part + (int64_t)(h->batch * h->nquad) * a.nbands * pk::kMaxK);
  a.values = values;
  a.rows = rows;
  a.cols = cols;
  a.k = k;
  a.planes = (int)(h->batch * h->nquad);
  const dim3 g1((unsigned)a.nbands, (unsigned)a.planes), g2((unsigned)((a.planes + pk::kWarps - 1) / pk::kWarps));
  const cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(a.thr, 0, (size_t)a.planes * sizeof(uint64_t), st) != cudaSuccess) return FHT_ERR_CUDA;
  // 16-byte columns when every row start is 16-byte aligned and W is a multiple of 4
  const bool vec = a.W % 4 == 0 && a.W >= 4 && aligned16(h->data) && a.rstride % 4 == 0 && a.qstride % 4 == 0 &&
                   a.bstride % 4 == 0;
  if (h->dtype == FHT_F32) {
    if (vec) pk::k_peaks_band4<float><<<g1, pk::kWarps * 32, 0, st>>>(a);
    else pk::k_peaks_band<float><<<g1, pk::kWarps * 32, 0, st>>>(a);
    pk::k_peaks_merge<float><<<g2, pk::kWarps * 32, 0, st>>>(a);
  } else {
    if (vec) pk::k_peaks_band4<int><<<g1, pk::kWarps * 32, 0, st>>>(a);
    else pk::k_peaks_band<int><<<g1, pk::kWarps * 32, 0, st>>>(a);
    pk::k_peaks_merge<int><<<g2, pk::kWarps * 32, 0, st>>>(a);
  }
  if (cudaGetLastError() != cudaSuccess) return FHT_ERR_CUDA;
  return 2;
}

int fht_cell_segment(const fht_hough* h, int64_t slot, int64_t row, int64_t col, fht_segment* out) {
  if (!h || !out) return FHT_ERR_ARG;
  if (row < 0 || row >= h->rows || col < 0 || col >= h->cols || slot < 0 || slot >= h->nquad) return FHT_ERR_ARG;
  int q;
  int64_t s;
  int64_t n;
  if (h->mode == FHT_MODE_QUADRANT) {
    q = h->quadrant;
    s = row;
    n = h->rows;
  } else if (h->mode == FHT_MODE_FULL) {
    if (h->layout == FHT_LAYOUT_QUADS) {
      q = (int)slot;
      s = row + h->row0;  // a shard's band starts at shift row0
    } else {  // CONCAT: P:111-113 thresholds, a shared row belongs to the earlier quadrant (R8)
      const int64_t Hp = h->Hp, Wp = h->Wp;
      if (row < Hp) { q = FHT_QA; s = Hp - 1 - row; }
      else if (row < 2 * Hp - 1) { q = FHT_QB; s = row - (Hp - 1); }
      else if (row < 2 * Hp - 2 + Wp) { q = FHT_QC; s = Wp - 1 - (row - (2 * Hp - 2)); }
      else { q = FHT_QD; s = row - (2 * Hp + Wp - 3); }
    }
    n = q >= 2 ? h->Wp : h->Hp;
  } else {
    return FHT_ERR_UNSUPPORTED;  // RANGE: the resampled frame has no single-pixel inverse
  }
  const bool tr = q >= 2;
  const int sigma = (q == FHT_QA || q == FHT_QD) ? 1 : -1;
  const int64_t fh = tr ? h->w : h->h, fw = tr ? h->h : h->w, W = h->cols;
  fht_segment sg{};
  sg.quadrant = q;
  sg.s = (int32_t)s;
  if (s < n) {
    // P:71 step 1: frame column (x0 + sigma*D_s(y)) of frame row y; P:73-77 step 2: mod W, keep the
    // original frame (QC/QD frames are the transposed image)
    const int K = ilog2(n);
    for (int64_t y = 0; y < fh && y < n; ++y) {
      int64_t xf = (col + sigma * (int64_t)dyadic_offset(K, (int)s, (int)y)) % W;
      if (xf < 0) xf += W;
      if (xf >= fw) continue;
      const int64_t px = tr ? y : xf, py = tr ? xf : y;
      if (sg.npix == 0) {
        sg.x0 = px;
        sg.y0 = py;
      }
      sg.x1 = px;
      sg.y1 = py;
      ++sg.npix;
    }
  }
  *out = sg;
  return FHT_OK;
}

}  // extern "C"
