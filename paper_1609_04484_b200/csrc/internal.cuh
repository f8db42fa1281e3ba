// internal.cuh -- private structures of libbie.so (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>
#include <string>
#include <vector>

#include "../../include/bie.h"

// ---------------------------------------------------------------------------
// Checked build (-DBIE_CHECKED, lib/libbie_checked.so): the
// stand-in for compute-sanitizer, which this GPU pool does not allow.  Every
// device allocation of the library gets 256-byte canary regions on both sides
// and is filled with 0xFF bytes (a NaN in every double, so a read of memory
// no kernel wrote propagates into the parity checks); bie_debug_check()
// verifies all live canaries, and freeing checks the block's own.  Kernels
// carry BIE_DCHECK(index bounds) on their global stores; a failed check
// records its source line in a device flag that bie_debug_check() reports.
// ---------------------------------------------------------------------------
namespace bie {
cudaError_t chk_malloc(void **p, size_t bytes, cudaStream_t st, bool async);
cudaError_t chk_free(void *p, cudaStream_t st, bool async);
}  // namespace bie
#ifdef BIE_CHECKED
template <class T>
static inline cudaError_t bie_chk_cudaMalloc(T **p, size_t b) {
    return ::bie::chk_malloc(reinterpret_cast<void **>(p), b, nullptr, false);
}
template <class T>
static inline cudaError_t bie_chk_cudaMallocAsync(T **p, size_t b, cudaStream_t st) {
    return ::bie::chk_malloc(reinterpret_cast<void **>(p), b, st, true);
}
#define cudaMalloc(p, b) bie_chk_cudaMalloc((p), (b))
#define cudaMallocAsync(p, b, st) bie_chk_cudaMallocAsync((p), (b), (st))
#define cudaFree(p) ::bie::chk_free((void *)(p), nullptr, false)
#define cudaFreeAsync(p, st) ::bie::chk_free((void *)(p), (st), true)
// per translation unit: first failing line of a device-side check
static __device__ int bie_dcheck_line = 0;
#define BIE_DCHECK(cond)                                          \
    do {                                                          \
        if (!(cond)) atomicCAS(&bie_dcheck_line, 0, __LINE__);   \
    } while (0)
#define BIE_DCHECK_TU(name)                                                            \
    namespace bie {                                                                    \
    int dcheck_##name() {                                                              \
        int h = 0;                                                                     \
        cudaMemcpyFromSymbol(&h, bie_dcheck_line, sizeof(int));                        \
        return h;                                                                      \
    }                                                                                  \
    }
#else
#define BIE_DCHECK(cond) \
    do {                 \
    } while (0)
#define BIE_DCHECK_TU(name)                  \
    namespace bie {                          \
    int dcheck_##name() { return 0; }        \
    }
#endif

namespace bie {

constexpr double kPi = 3.14159265358979323846;
constexpr uint32_t kGeomMagic = 0x4745304du;   // "GEOM"
constexpr uint32_t kBlockMagic = 0x424c4b44u;  // "BLKD"
// internal operator bit of dlp_apply_impl's flags: the single-layer operator with
// the Kapur-Rokhlin correction (NEXT-1) instead of the completed DLP
constexpr unsigned kOpSLP = 1u << 16;

void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);
#define BIE_CUDA_TRY(expr)                                          \
    do {                                                            \
        cudaError_t _e = (expr);                                    \
        if (_e != cudaSuccess) return ::bie::cuda_fail(_e, #expr);  \
    } while (0)
#define BIE_RC_TRY(expr)                \
    do {                                \
        const int _rc = (expr);         \
        if (_rc != BIE_OK) return _rc;  \
    } while (0)

// Static, perfectly balanced partition of the (target-block x source-tile)
// work units of the all-pairs kernel over a persistent grid.
struct PairSched {
    int nv = 0;         // vectors per launch (template variant)
    int R = 0;          // targets per thread
    int TS = 0;         // sources per smem tile
    int TB = 0;         // targets per CTA tile (= threads * R)
    int nTB = 0, nTS = 0;
    long long U = 0;    // nTB * nTS units
    int P = 0;          // persistent CTAs
    int S = 0;          // max partial slots per target block
    int smem = 0;
    long long Useg = 1; // units per dynamically claimed segment
};

struct BlockDiag;
// What a captured GMRES iteration graph depends on (gmres.cu): the operator, the
// BD handle (pointer + serial, so a new factorisation at a reused address
// does not match), tol, max_iter and every buffer the body's kernels address.
struct GmGraphKey {
    const BlockDiag *bd = nullptr;
    unsigned long long bd_serial = 0;
    unsigned opf = 0;
    int max_iter = 0;
    double tol = 0.0;
    const void *V = nullptr, *w = nullptr, *small = nullptr, *partial = nullptr, *gpartial = nullptr,
               *slp_s = nullptr;
    bool operator==(const GmGraphKey &o) const {
        return bd == o.bd && bd_serial == o.bd_serial && opf == o.opf && max_iter == o.max_iter && tol == o.tol &&
               V == o.V && w == o.w && small == o.small && partial == o.partial && gpartial == o.gpartial &&
               slp_s == o.slp_s;
    }
};

// GMRES workspace cached on the geometry (grow-only): per-call cudaMalloc /
// cudaMallocHost left the device idle for up to ~1 s in some steps.
struct GmresWork {
    double *V = nullptr, *w = nullptr, *t = nullptr, *H = nullptr, *small = nullptr, *partial = nullptr;
    size_t V_cap = 0, n_cap = 0, H_cap = 0, small_cap = 0, partial_cap = 0;
    double *pinned = nullptr;  // 8 + 2 * 8 doubles
    cudaEvent_t evs[8] = {};
    // bie_gmres_solve*: the captured iteration loop (conditional WHILE graph)
    cudaStream_t cap = nullptr;  // private capture stream
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t gexec = nullptr;
    GmGraphKey gkey;
    long long body_launches = 0;  // kernels per iteration of the graph body
    bool graph_off = false;       // capture failed once: host-enqueued loop from then on
};

struct Geometry {
    uint32_t magic = kGeomMagic;
    int N = 0, M = 0, n_pore = 0, n_outer = 0;
    int wall_lo = 0;          // first Gamma_0 node (= M * n_pore)
    // node table (device, SoA)
    double2 *pos = nullptr;   // x_j
    double2 *nw = nullptr;    // w_j n_j / pi (folded DLP source weight)
    double2 *nrm = nullptr;   // n_j
    double2 *tan = nullptr;   // t_j
    double *w = nullptr;      // w_j
    double *selfc = nullptr;  // w_j kappa_n,j / (2 pi)
    double *kappa = nullptr;  // kappa_n,j = x''.n / |x'|^2
    double4 *pore = nullptr;  // (cx, cy, r, |Gamma_k|)
    double wall_len = 0.0;    // |Gamma_0|
    // host copies needed for scheduling / BD
    std::vector<double> h_pore_r;
    // workspace
    double *partial = nullptr;  // [S][nvec<=16][2N]
    size_t partial_elems = 0;
    double *moments = nullptr;  // [16][M][3] (lambda_x, lambda_y, mu) + [16] nu
    double *stage_in = nullptr, *stage_out = nullptr;  // e2e staging [16][2N] each
    PairSched sched[5];         // nv = 1, 2, 4, 8, 16
    int occ[5] = {0, 0, 0, 0, 0};  // resident pair CTAs per SM per variant
    // single-layer operator (NEXT-1)
    PairSched sched_slp[5];
    int occ_slp[5] = {0, 0, 0, 0, 0};
    double kr[6] = {0, 0, 0, 0, 0, 0};  // Kapur-Rokhlin gamma_1..gamma_6 (reading C24)
    double *slp_s = nullptr;             // [16][2N] S = w sigma / (4 pi) (lazy)
    int num_sms = 0;
    // symmetric nvec = 1 path (lazily allocated; see dlp.cu)
    int sym_state = 0;            // 0 = not prepared, 1 = ready, -1 = unavailable (memory cap)
    double4 *sym_Q = nullptr;     // [N] per-node quadratic forms
    long long *sym_off = nullptr; // [nTB + 1] unit prefix per 512-node block
    unsigned long long *sym_acc = nullptr;  // [3][2N] fixed-point limbs of the pair sums (dlp.cu fx_add)
    int sym_occ[2] = {1, 1};      // resident CTAs per SM of the DLP / SLP symmetric kernel
    double *sym_diag = nullptr;   // [2N]
    cudaStream_t side = nullptr;  // in-block kernel beside the pair kernel (fork/join by events)
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // BD factor lookahead (blockdiag.cu): high-priority panel stream and its events, created on
    // first use and kept (a fresh priority stream per factor showed host-side stalls of 0.1-0.7 s)
    cudaStream_t bd_hp = nullptr;
    cudaEvent_t bd_ev[3] = {nullptr, nullptr, nullptr};
    int sym_nTB = 0, sym_P = 0, sym_variant = 0;  // (8, 2, 2), lockstep groups of 4, 6 CTAs/SM: fastest measured
    int slp_sym_variant = 0;  // (8, 2, 2): fastest measured
    unsigned long long *sym_trace = nullptr;  // BIE_SYM_TRACE: per-CTA start/end times of the last launch
    unsigned long long *sym_counter = nullptr;  // [0] dynamic segment counter, [1] max |Q| bits (accumulation window)
    unsigned long long *pair_counter = nullptr; // [8] counters of the one-sided launches of one apply
    long long sym_Useg = 1;                     // units per segment
    int sym_dsplit = 1;                         // source split of the in-block kernel (small N)
    long long sym_U = 0;
    GmresWork gm;               // bie_gmres_solve* workspace
    GmresWork gmb;              // bie_gmres_solve_batch* workspace (w holds Win | Wt | Wout)
    // profiling (bie_profile_begin/end): 4 events per recorded apply
    bool prof = false;
    std::vector<cudaEvent_t> prof_ev;
    size_t prof_used = 0;
};

// process-wide count of kernels launched by the library (bie_launch_count)
void count_launch(int n = 1);

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL) for the kernels of one GMRES iteration
// (matvec, BD apply, Krylov kernels; DESIGN.md s5 GMRES).  Each such kernel
// starts with pdl_wait() (griddepcontrol.wait: blocks until the preceding grid
// has completed and its memory is visible; a no-op for a normal launch), and
// launch_pdl() lets the next grid be scheduled while this one drains, so the
// launch latency between the ~20 short kernels of a small-N iteration overlaps
// the previous kernel's tail.  Every kernel launched this way waits before it
// touches memory, so completion stays transitive along the stream.
// BIE_PDL=0 disables it (A/B).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    (void)cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);  // error -> cudaGetLastError()
}
#define BIE_LAUNCH(kern, grid, block, smem, st, ...) \
    ::bie::launch_pdl(kern, dim3(grid), dim3(block), (size_t)(smem), (st), __VA_ARGS__)

unsigned long long next_bd_serial();
struct BlockDiag {
    uint32_t magic = kBlockMagic;
    unsigned long long serial = next_bd_serial();  // distinguishes factorisations (GMRES graph cache)
    Geometry *g = nullptr;
    int b0 = 0, b1 = 0;             // body range [b0, b1) (pores 0..M-1, wall M)
    int op = 0;                     // 0: blocks of the completed DLP; 1: of the SLP (NEXT-1)
    int row_lo = 0, row_hi = 0;     // node range covered; apply vectors are local [2 (row_hi-row_lo)]
    int nb = 0;                     // number of bodies
    std::vector<int> lo, n;         // node range per body
    std::vector<long long> off;     // offset of body b's inverse (doubles)
    double *inv = nullptr;          // explicit inverses, row-major [2n_b][2n_b]
    long long *d_off = nullptr;
    int *d_lo = nullptr, *d_n = nullptr;
    // structured pore blocks (NEXT-4, bie_blockdiag_factor_structured): inv/off then
    // hold only the wall; pores use X = B_ref^-1 plus a rank-2 Woodbury term each
    int structured = 0;
    double *sX = nullptr;           // [2n_p][2n_p] inverse of the reference pore block
    double *sW = nullptr;           // [2n_p][2]   W = X U
    double *sG = nullptr;           // [4]         G = U^T X U
    double *sM = nullptr;           // [M][4]      M_k = c_k (I + c_k G)^-1
    std::vector<double> h_M;        // host copy of M_k
    // structured == 2: SLP pore blocks as block-circulant matrices in the
    // rotating frame (bie_blockdiag_factor_structured_slp, blockdiag.cu)
    double *sD = nullptr;           // [M][n_p][4]  first block row d_k(m) of the rotating-frame inverse
    double2 *sTmpl = nullptr;       // [n_p]        (cos, sin)(2 pi j / n_p), the pore node angles
};

Geometry *as_geom(bie_geometry_t g);
BlockDiag *as_bd(bie_blockdiag_t b);

// geometry.cu
void kr_weights(double gamma[6]);
void pore_template(int n, std::vector<double2> &out);  // correctly rounded (cos, sin)(2 pi j / n), reading C27
// dlp.cu
int dlp_apply_impl(Geometry *g, const double *sigma, double *out, int nvec, unsigned flags, int row_begin,
                   int row_end, cudaStream_t s);
int build_schedules(Geometry *g);
// blockdiag.cu
int blockdiag_apply_impl(BlockDiag *bd, const double *in, double *out, int nvec, cudaStream_t s);
// geometry.cu: the side stream and fork/join events of g (created on first use)
int ensure_side_stream(Geometry *g);
// gmres.cu kernels used by other units
}  // namespace bie
