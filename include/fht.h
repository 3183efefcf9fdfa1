/*
 * fht.h -- C ABI of libfht.so: the Brady dyadic Fast Hough Transform on one B200 (sm_100a),
 * as studied in M. Aliev, E.I. Ershov, D.P. Nikolaev, "On the use of FHT, its modification for
 * practical applications and the structure of Hough image" (arXiv 1811.06378).
 *
 * Citations: P:n = PAPER.md line n (section in brackets); S:n = SPEC.md line n.
 * Readings R1..R26 are listed in DESIGN.md ("Readings of the paper").
 *
 * Conventions common to every call
 * --------------------------------
 *  - Every buffer pointer in fht_image / fht_hough and every workspace pointer is a DEVICE
 *    pointer allocated and owned by the caller. The library allocates no device memory, keeps
 *    no global mutable state (beyond a per-device record of which kernels have had their dynamic
 *    shared-memory limit raised) and retains no pointer after a call returns. All device work is
 *    enqueued on `stream` (0 = legacy default stream); buffers must stay alive until it ends.
 *  - Strides are in ELEMENTS. Pointers must be aligned to their element size (FHT_ERR_ALIGN
 *    otherwise). Output descriptors from fht_hough_describe() have 16-byte row pitches; the
 *    kernels pick 128-bit vector accesses where base pointers and pitches allow them.
 *  - Argument errors are detected synchronously, before anything is enqueued, and reported as
 *    a negative fht_status; nothing is thrown across the ABI. On success the compute calls
 *    (fht_quadrant, fht_full, fht_angle_range, fhtshift) return the number (>= 1) of kernels
 *    they enqueued; the host-only calls return FHT_OK (0). A launch failure returns
 *    FHT_ERR_CUDA; device faults surface at the caller's next synchronisation.
 *  - Element types: input u8, i32 or f32. Output is i32 for u8/i32 input (exact; the caller
 *    owns i32 overflow), f32 for f32 input (IEEE round-to-nearest adds, R21 tolerance).
 *  - Coordinates: x = column (right), y = row (down). A Hough cell is (s, x0): s = shift
 *    row, x0 = column in the cyclic layout of width W ("mod(w + h)").
 *  - Quadrants (R4): QA = (I, +), QB = (I, -), QC = (I^T, -), QD = (I^T, +) where
 *    (image, sigma) means H[s][x0] = sum_y Ipad[y][(x0 + sigma * D_{Hp,s}(y)) mod W] and
 *    D is the dyadic pattern of S:71 (R1). QC/QD use the transposed image by index
 *    transposition -- no copy is made. Ipad is the image zero-extended to Hp = next_pow2(rows)
 *    rows (R3) and W = cols + Hp columns ("(w + h) x h").
 */
#ifndef FHT_H
#define FHT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* fht_stream_t; /* == cudaStream_t */

typedef enum {
  FHT_OK = 0,
  FHT_ERR_ARG = -1,         /* bad scalar argument, NULL pointer, aliasing, bad angle range */
  FHT_ERR_DTYPE = -2,       /* dtype not supported for this call / output dtype mismatch */
  FHT_ERR_SHAPE = -3,       /* output descriptor shape does not match the transform */
  FHT_ERR_ALIGN = -4,       /* pointer or row pitch not 16-byte aligned */
  FHT_ERR_UNSUPPORTED = -5, /* valid request the GPU path does not implement (e.g. pad != Hp) */
  FHT_ERR_WORKSPACE = -6,   /* workspace NULL or smaller than fht_workspace_bytes() */
  FHT_ERR_STATE = -7,       /* fhtshift on an already shifted descriptor */
  FHT_ERR_CUDA = -8         /* a CUDA launch or runtime call failed */
} fht_status;

typedef enum { FHT_U8 = 0, FHT_I32 = 1, FHT_F32 = 2 } fht_dtype;
typedef enum { FHT_QA = 0, FHT_QB = 1, FHT_QC = 2, FHT_QD = 3 } fht_quadrant_id;
typedef enum { FHT_MODE_QUADRANT = 0, FHT_MODE_FULL = 1, FHT_MODE_RANGE = 2 } fht_mode;
/* QUADS: [batch][4][Pmax][W] unflipped quadrant images (BASELINE C2 "four quadrants").
 * CONCAT: [batch][2(Hp+Wp)-3][W], P:89 order "QA flipped; QB; QC flipped; QD", a row shared by
 * two neighbours written once by the earlier quadrant (R8). */
typedef enum { FHT_LAYOUT_QUADS = 0, FHT_LAYOUT_CONCAT = 1 } fht_layout;

/* Input image batch: element (b, y, x) at data[b*batch_stride + y*row_stride + x]. */
typedef struct {
  const void* data;
  int32_t dtype; /* fht_dtype */
  int32_t _pad0;
  int64_t batch, h, w;
  int64_t batch_stride, row_stride;
} fht_image;

/* §4 plan (R12-R17). theta = inclination from vertical, tan(theta) = dx/dy.
 * Lines with slope k in [k_lo, k_hi] are sheared by k_lo and scaled by alpha = 1/(k_hi-k_lo)
 * onto QA's slopes [0, 1] (scale law P:124, shear law P:132, composition P:144).
 * Transformed row y (never materialised):
 *   T(x', y) = I[y][colmap[x' - e_y]] if 0 <= x' - e_y < w_content, else 0   (unwrapped x')
 *   e_y = floor(g*y + 0.5), g = alpha*(-k_lo);  colmap[u] = min(w-1, floor((u+0.5)/alpha)).
 * Output: Hp rows x W cyclic columns, W = w_content + max(Hp, 1 + max_s spread_s) (R17). */
typedef struct {
  double theta_min_deg, theta_max_deg;
  double k_lo, k_hi, alpha, g;
  int64_t h, w, Hp;
  int64_t w_content; /* w' = ceil(alpha*w) */
  int64_t W;         /* W' */
  int64_t e_min, e_max; /* min / max of e_y over y < h */
  int64_t rows;         /* output rows: Hp (fht_angle_plan), S_max + 1 (fht_angle_plan_make_pruned) */
  int64_t transposed;   /* 1: mostly-horizontal plan -- the frame is the transposed image and h, w
                           above are the FRAME's (image w, h); angles are measured from horizontal */
} fht_angle_plan_t;

/* Output (Hough image) descriptor. Fill it with fht_hough_describe(), then set `data`. */
typedef struct {
  void* data;
  int32_t dtype;    /* I32 for integer input, F32 for float input */
  int32_t mode;     /* fht_mode */
  int32_t layout;   /* fht_layout (FULL mode only) */
  int32_t shifted;  /* 1 = rows hold the fhtshift-ed image (§5); set by the library */
  int32_t quadrant; /* QUADRANT mode: which quadrant */
  int32_t _pad0;
  int64_t batch, nquad, rows, cols;       /* nquad = 4 for FULL/QUADS, else 1 */
  int64_t batch_stride, quad_stride, row_stride;
  int64_t h, w, Hp, Wp;                   /* source image dims; Hp/Wp = padded powers of two */
  fht_angle_plan_t plan;                    /* valid iff mode == RANGE */
  int64_t row0;     /* a row band of a sharded transform (fht_shard_describe): row r holds shift row0 + r */
} fht_hough;

/* Optional per-call execution options (may be NULL).
 *  events: caller-created CUDA events (cudaEvent_t cast to void*); when non-NULL the call records
 *    events[i] on the launching stream right before its i-th kernel launch and events[n] right
 *    after its last (n = the call's return value), for i < n_events. Used by bench.py to time
 *    each kernel.
 *  aux_stream: a second caller-owned stream (cudaStream_t, != stream) or NULL. When the batch is
 *    processed in several scratch chunks, pass 1 of chunk k+1 runs on aux_stream concurrently
 *    with pass 2 of chunk k on `stream` (two scratch buffers, ordered by events). The call is
 *    still complete when `stream` reaches it; aux_stream is left with no pending work the caller
 *    must wait for. fht_workspace_bytes() already includes the second buffer. */
typedef struct {
  void* const* events;
  int32_t n_events;
  int32_t _pad0;
  void* aux_stream;
} fht_exec_opts;

/* Fill `out` (except `data`) with the contiguous shape of the transform of `img`:
 *   QUADRANT: rows = Hp, cols = W = w + Hp (QA/QB) or Wp rows, h + Wp cols (QC/QD);
 *   FULL/QUADS: nquad 4, rows = max(Hp, Wp), cols = Hp + Wp (R9);
 *   FULL/CONCAT: rows = 2(Hp+Wp)-3, cols = Hp + Wp;
 *   RANGE: rows = plan->Hp, cols = plan->W.
 * `plan` may be NULL unless mode == RANGE. Returns FHT_OK or a negative fht_status. */
int fht_hough_describe(int mode, int layout, int quadrant, const fht_image* img,
                       const fht_angle_plan_t* plan, fht_hough* out);

/* Quadrant-mode descriptor with a pad other than Hp (R22): cols = w_frame + pad_cols
 * (w_frame = w for QA/QB, h for QC/QD); pad_cols = -1 means Hp (= fht_hough_describe). */
int fht_hough_describe_pad(int quadrant, const fht_image* img, int64_t pad_cols, fht_hough* out);

/* Workspace for fht_quadrant with this pad (a pad below h_frame - 1 adds the pad = Hp image). */
size_t fht_quadrant_workspace_bytes(const fht_image* img, int quadrant, int64_t pad_cols);

/* Device workspace (bytes) the call needs for `img` (pass-1 scratch + tables). */
size_t fht_workspace_bytes(int mode, const fht_image* img, const fht_angle_plan_t* plan);

/* Output pair of the transform calls below. `out` receives the Hough image H; `out_shifted`
 * receives fhtshift(H) (§5), written by the same pass-2 kernel from the same
 * registers (no re-read of H). Either may be NULL, not both; both must be described by
 * fht_hough_describe() for the same transform, with `data` set, 16-byte aligned base and row
 * pitch, and must not overlap each other, the image or the workspace. On success
 * out->shifted = 0 and out_shifted->shifted = 1. */

/* One quadrant. pad_cols: -1 (= Hp) or any pad >= 0 (R22). For pad >=
 * h_frame - 1 (h_frame = h for QA/QB, w for QC/QD; the paper's literal "extended by h" included)
 * every line's columns stay apart mod w_frame + pad and the two passes write the image directly;
 * a smaller pad folds lines cyclically ("mod(w+h)"): the pad = Hp transform goes into the
 * workspace and one more kernel folds it mod w_frame + pad. Outputs from
 * fht_hough_describe_pad(quadrant, img, pad_cols, ...); workspace fht_quadrant_workspace_bytes(). */
int fht_quadrant(const fht_image* img, int quadrant, int64_t pad_cols, fht_hough* out,
                 fht_hough* out_shifted, void* ws, size_t ws_bytes, fht_stream_t stream,
                 const fht_exec_opts* opts);

/* Full four-quadrant transform. `layout` must equal the outputs' layout. */
int fht_full(const fht_image* img, int layout, fht_hough* out, fht_hough* out_shifted, void* ws,
             size_t ws_bytes, fht_stream_t stream, const fht_exec_opts* opts);

/* Host-only: build the §4 plan (P:124 scale law, P:132 shear law, P:144 composition) for an h x w
 * image and inclinations [theta_min, theta_max] (degrees from vertical, R12). FHT_ERR_ARG if
 * theta_min >= theta_max, |theta| >= 90 deg, or alpha*w < 1; FHT_ERR_UNSUPPORTED for h > 4096.
 * Deterministic double arithmetic, no FMA (R16). O(Hp log Hp) host work: W' (R17) takes the
 * per-row spread of e_y - D_s(y) from the FHT block recursion with (min, max) in place of +. */
int fht_angle_plan(int64_t h, int64_t w, double theta_min_deg, double theta_max_deg, fht_angle_plan_t* out);

/* Host-only: the inclination (degrees; from vertical, or from horizontal for a transposed plan) of
 * the lines row s of a range output holds (R19, "shift = h tg(phi)"): row s's patterns have
 * endpoint slope s/(Hp-1) in the transformed frame; undoing the scale and shear gives
 * tan = k_lo + s / (alpha (Hp - 1)). Row 0 is theta_min; row Hp-1 of a §4 plan is theta_max.
 * FHT_ERR_ARG for NULL pointers or s outside [0, Hp). */
int fht_angle_of_row(const fht_angle_plan_t* plan, int64_t s, double* deg);

/* Shift-range-pruned plan (north_star "computes only the stages and shift ranges
 * the restriction needs"): shear only (alpha = 1, w' = w, colmap = identity,
 * e_y = floor(-k_lo*y + 0.5)), so the slopes [k_lo, k_hi] become QA rows s = (k - k_lo)*(Hp-1) of
 * the sheared image and only rows s <= S_max = ceil((k_hi - k_lo)*(Hp-1)) are computed and stored
 * (plan.rows = S_max + 1 <= Hp). W' follows R17 with the spread taken over those rows. Requires
 * k_hi - k_lo <= 1 (otherwise FHT_ERR_UNSUPPORTED: use fht_angle_plan's scaled frame); other
 * errors as fht_angle_plan. fht_angle_range_plan computes a pruned plan on the v2 kernels only
 * (FHT_ERR_UNSUPPORTED for the degenerate frames of the v1 path). */
int fht_angle_plan_make_pruned(int64_t h, int64_t w, double theta_min_deg, double theta_max_deg,
                               fht_angle_plan_t* out);

/* General plan (SURVEY §8(f) f4 "mostly-horizontal range"). flags: FHT_PLAN_PRUNED (as
 * fht_angle_plan_make_pruned) and/or FHT_PLAN_HORIZONTAL: the range is of inclinations from the
 * HORIZONTAL (tan = dy/dx) and the plan is built on the transposed image, the frame of the
 * mostly-horizontal quadrants QC/QD -- so a range near horizontal keeps alpha near 1
 * instead of being squeezed by the vertical frame's scale. Horizontal [0, 45] equals QD exactly,
 * [-45, 0] QC with rows reversed. h, w are the IMAGE's; the plan stores the frame's (swapped).
 * Errors as fht_angle_plan / fht_angle_plan_make_pruned. */
enum { FHT_PLAN_PRUNED = 1, FHT_PLAN_HORIZONTAL = 2 };
int fht_angle_plan_make_ex(int64_t h, int64_t w, double theta_min_deg, double theta_max_deg, int32_t flags,
                           fht_angle_plan_t* out);

/* Angle-range-restricted transform (§4, "perform a transform for an arbitrary range of
 * angles [gamma1; gamma2]"): QA of the virtually sheared+scaled image, the shear and
 * scale fused into the first FHT iteration (pass-1 loader). f32/u8/i32 input. The §4 plan of
 * (img->h, img->w, theta_min, theta_max) is built inside the call (fht_angle_plan); the outputs
 * must be described with that plan (fht_hough_describe(FHT_MODE_RANGE, ..., &plan, ...)), else
 * FHT_ERR_SHAPE. Workspace: fht_angle_range_workspace_bytes(). Errors as fht_angle_plan plus the
 * output / workspace errors of the other transform calls. Returns the kernels enqueued (3). */
int fht_angle_range(const fht_image* img, double theta_min_deg, double theta_max_deg, fht_hough* out,
                    fht_hough* out_shifted, void* ws, size_t ws_bytes, fht_stream_t stream,
                    const fht_exec_opts* opts);
size_t fht_angle_range_workspace_bytes(const fht_image* img, double theta_min_deg, double theta_max_deg);

/* The same transform for a prepared plan: a §4 plan, a shift-range-pruned plan or a mostly-
 * horizontal plan (fht_angle_plan_make_pruned / _ex). Workspace: fht_workspace_bytes(FHT_MODE_RANGE,
 * img, plan). */
int fht_angle_range_plan(const fht_image* img, const fht_angle_plan_t* plan, fht_hough* out,
                         fht_hough* out_shifted, void* ws, size_t ws_bytes, fht_stream_t stream,
                         const fht_exec_opts* opts);

/* §5 fhtshift (R11): out[r][x] = in[r][(x - k_r) mod cols] with R11's generic rule
 * k = ceil((W - len_s)/2) - start_s, which centres row s's meaningful run: for quadrants
 * len_s = w_frame + s, so k_r = ceil((pad+s)/2) for sigma=+1 and ceil((pad-s)/2) for sigma=-1 with
 * pad = cols - w_frame (= n, the row count, in FULL mode and for the default quadrant pad); RANGE
 * mode takes (start_s, len_s) from the row's support. `in` must be unshifted (FHT_ERR_STATE otherwise); `out` must have the same shape and
 * not alias `in`; on success out->shifted = 1. Bit copy: exact for every dtype. One kernel: a warp
 * per row, 16-byte loads/stores when cols, every stride and both bases are 16-byte aligned; in RANGE
 * mode each block first reduces its rows' support (start_s, len_s) from an e_y table in shared
 * memory. Allocates nothing. Returns 1 (kernels enqueued). */
int fhtshift(const fht_hough* in, fht_hough* out, fht_stream_t stream);

/* ---- Single-image sharding over ranks ------------------------------------------
 * The full transform (FULL/QUADS; square frames, Hp == Wp) split over `world` GPUs, one process per
 * GPU. With the pass split K = m + L of the frame, rank g runs pass 1 (levels 1..m) on
 * its strips i in [g S, (g+1) S), S = 2^L / world -- image rows [g Hp/world, (g+1) Hp/world) of QA/QB
 * and image columns of QC/QD -- and sends the shifts j of rank h's groups J_h = [h J, (h+1) J),
 * J = 2^m / world, to rank h; rank h runs pass 2 (levels m+1..K) on J_h, which yields output rows
 * t in [h Hp/world, (h+1) Hp/world) of every quadrant (t = j 2^L + u), a row band. Pass 2 of group j
 * needs F_m[i][j] of EVERY strip i (the pre-shear identity), so the exchange between the passes is ONE
 * all-to-all of the pass-1 scratch (Fig. 6 iteration; the multi-pass identity). The paper
 * has no multi-GPU content; this is the north_star's data-parallel path at a size beyond one GPU.
 *
 * Buffers (device, caller-owned, all ranks the same sizes): rank g's chunk for rank h is
 * [z = image * 4 + quadrant][j_local < J][strip_local < S][pitch] elements of the scratch type (u16 for
 * u8 input, else the accumulator), chunk_bytes each; a receive buffer is world chunks, chunk g from
 * rank g. Requires world a power of two <= 8 that divides 2^m and 2^L (FHT_ERR_UNSUPPORTED otherwise). */
typedef struct {
  int32_t world, rank;
  int32_t m, L;              /* the frame's pass split (K = m + L) */
  int64_t S, J;              /* strips and groups per rank */
  int64_t rows_per_rank;     /* Hp / world: rows of this rank's output band */
  int64_t pitch;             /* scratch row pitch, elements */
  int32_t scratch_es, _pad0; /* scratch element bytes */
  int64_t chunk_rows;        /* batch * 4 * J * S */
  int64_t chunk_bytes;       /* one chunk (16-byte multiple) */
  int64_t send_bytes, recv_bytes;  /* world * chunk_bytes */
  fht_hough band;            /* this rank's output band: FULL/QUADS, rows = Hp/world, row0 = rank Hp/world */
} fht_shard;

/* Host-only: the geometry above for `img` (data may be NULL). */
int fht_shard_describe(const fht_image* img, int world, int rank, fht_shard* out);

/* Pass 1 of rank sh->rank. dst[h] (h < world, device pointers): where rank h's chunk goes -- either
 * this rank's send buffer + h * chunk_bytes (the caller then runs one all-to-all, e.g. NCCL), or rank
 * h's RECEIVE buffer + rank * chunk_bytes mapped into this process (peer memory over NVLink /
 * NVSwitch): the exchange then happens in pass 1's own TMA stores and no collective is needed. One
 * kernel; returns 1. */
int fht_shard_pass1(const fht_image* img, const fht_shard* sh, void* const* dst, fht_stream_t stream);

/* Pass 2 of rank sh->rank from its receive buffer (all world chunks present; the caller orders it
 * after every rank's pass 1 / the all-to-all). band / band_shifted: descriptors equal to sh->band with
 * `data` set (either may be NULL, not both); band_shifted receives the fhtshift-ed rows (§5, R11: the
 * shift of global row row0 + r). One kernel; returns 1. */
int fht_shard_pass2(const fht_image* img, const fht_shard* sh, const void* recv, fht_hough* band,
                    fht_hough* band_shifted, fht_stream_t stream);

/* Human-readable name of a status code (static string). */
const char* fht_status_string(int status);

/* ---- Peaks and line recovery ---------------------------------------------- */

/* Top-k peaks of every Hough plane (plane = image b, quadrant slot q; batch*nquad planes of
 * rows x cols; R25). A cell beats a neighbour when its value is larger, or equal and it
 * comes first in row-major order; a peak beats each of its up to 8 neighbours (columns cyclic:
 * x0 is taken mod W; rows not). The k (1..32) peaks with the largest values (ties: smaller
 * row-major index first) are written to values[plane*k + i] (the Hough dtype), rows[...] and
 * cols[...] (int32), all DEVICE pointers owned by the caller; a plane with fewer than k peaks pads
 * with row = col = -1, value 0. ws: fht_peaks_workspace_bytes(h) device bytes. Two kernels (a
 * streaming pass over bands of rows, a per-plane merge). Errors: ARG (k outside 1..32, NULL),
 * DTYPE, WORKSPACE, UNSUPPORTED (rows*cols >= 2^32, or more than 65535 planes). Returns 2 (kernels
 * enqueued). */
size_t fht_peaks_workspace_bytes(const fht_hough* h);
int fht_peaks(const fht_hough* h, int32_t k, void* values, int32_t* rows, int32_t* cols, void* ws,
              size_t ws_bytes, fht_stream_t stream);

/* The pattern of one Hough cell on the original image (§3.2 steps 1-2; CONCAT rows are
 * attributed by P:111-113, R8): frame column (col + sigma*D_s(y)) mod W of frame rows y < n, kept
 * where it lies inside the original frame (QC/QD: transposed). The kept pixels form one run;
 * out gets its first (x0, y0) and last (x1, y1) pixel in frame-row order and the pixel count npix
 * (0 = the cell is in the black zone), plus the quadrant and its shift s. Host-only,
 * no device access. QUADRANT and FULL descriptors (`slot` = the QUADS plane; 0 otherwise);
 * RANGE returns FHT_ERR_UNSUPPORTED. */
typedef struct {
  int32_t quadrant, s;
  int64_t npix;
  int64_t x0, y0, x1, y1;
} fht_segment;
int fht_cell_segment(const fht_hough* h, int64_t slot, int64_t row, int64_t col, fht_segment* out);

#ifdef __cplusplus
}
#endif
#endif /* FHT_H */
