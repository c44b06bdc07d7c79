// internal.h -- declarations shared by the library's translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstddef>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mlmc.h"

namespace mlmc {

// ---------------------------------------------------------------- host KL (host_kl.cpp)
struct KLModes {
    std::vector<int32_t> ik, jk;     // 1-based 1D mode indices
    std::vector<double> lam;         // 2D eigenvalues, descending (R11 tie-break)
    std::vector<double> w;           // 1D roots, w[i-1] belongs to 1D mode i
    std::vector<double> nrm;         // 1D normalisation constants
    double c = 0.0;                  // 1/corr_len
};
int kl_modes(double sigma2, double corr_len, int m, KLModes& out);
// Phi[p*m + k] for the 2N^2 triangle centroids of an N x N mesh (R10 ordering).
void build_phi(const mlmc_problem& pr, const KLModes& kl, int N, std::vector<double>& phi);
// Separable form of the same synthesis (both fields are sums of products f_a(x1) g_b(x2)): mode k =
// c_k f_{a_k}(x1) g_{b_k}(x2), the modes listed by x-function index a (CSR: aoff[K+1], mk = mode index,
// mb = b_k, mc = c_k), and per mesh the four tables tab[t][i][a] (t = 0: f at (i + 1/3) h, 1: f at
// (i + 2/3) h, 2: g at (i + 1/3) h, 3: g at (i + 2/3) h; i < N, a < K).
struct SepModes {
    int K = 0;
    std::vector<int32_t> aoff, mk, mb;
    std::vector<double> mc;
};
void build_sep_modes(const mlmc_problem& pr, const KLModes& kl, SepModes& out);
void build_sep_tables(const mlmc_problem& pr, const KLModes& kl, const SepModes& sm, int N, std::vector<double>& tab);

// ---------------------------------------------------------------- kernels
// K0: xi[b*m + k] ~ N(0,1), b < nb, for global index first_index + b.
cudaError_t launch_rng(double* xi, int m, uint64_t nb, uint64_t seed, int level, uint64_t first_index,
                       cudaStream_t s);
// K1+K2: a[b*P + p] = exp(sum_k xi[b*m+k] * phi[p*m+k]).  keys (optional, device, 2*nb u64, zeroed
// by the caller): keys[2b] = max_p a (bits), keys[2b+1] = ~min_p a (bits), the coefficient contrast.
cudaError_t launch_field(const double* phi, const double* xi, double* a, int P, int m, uint64_t nb,
                         unsigned long long* keys, cudaStream_t s);
// K1s: the same a_T from the separable form, a = exp(F W) with W = C_xi G^T (two small DMMA contractions
// per sample instead of the P x m one).  tab: the four 1D tables [4][N][K] (build_sep_tables); kmap / cmap
// (device, K x K): the mode k = (a, b) and its c_k, or -1 / 0 where no mode has that pair.
// order / done (optional, with keys; nb <= kOrderMax): the last CTA also writes the longest-first order of the
// batch (as launch_order would); done is a zeroed device counter.
cudaError_t launch_field_sep(const double* tab, const int* kmap, const double* cmap, int K, const double* xi,
                             double* a, int N, int m, uint64_t nb, unsigned long long* keys, cudaStream_t s,
                             int* order = nullptr, unsigned* done = nullptr);
bool field_sep_supported(int N, int K);   // N = 8, 16 or a multiple of 32; K <= 32
bool field_use_dense();   // MLMC_FIELD_KERNEL=dense|ffma selects the P x m synthesis (A/B)
bool field_force_sep();   // MLMC_FIELD_KERNEL=sep selects the separable synthesis on every mesh (tests)
// Longest-first order of nb <= kOrderMax systems by descending contrast max a / min a (a single-CTA
// bitonic sort of the field keys): order[i] = system index.  The contrast predicts the MINRES
// iteration count (correlation 0.83 on configs[1] level 3), so the job counter hands out the long
// solves first (LPT scheduling of the persistent CTAs).
constexpr int kOrderMax = 8192;
constexpr int kOrderMinN = 16;   // (tuning build: MLMC_ORDER_MIN_N overrides in use_order)
constexpr size_t kOrderScratch = 4 * kOrderMax + 4 * 512 + 4 * 64;   // bytes of shared memory the order needs
cudaError_t launch_order(const unsigned long long* keys, int nb, int* order, cudaStream_t s);
// K3: MINRES for nb systems on the N x N mesh; writes out[b*8 + {0,2,4,6} + slot].  order (optional,
// device, nb ints): the sequence in which the systems are taken (order_kernel: longest first).
cudaError_t launch_minres(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out,
                          int slot, unsigned* job_counter, bool verify, const int* order, cudaStream_t s,
                          int xmode = 0, double* xio = nullptr);
bool minres_supported(int N);
// K3 v2 (k_minres_tile.cu): 2-column register tiles for N = 8, 16, 32, 64; variant < 0 = not used for N.
int minres_tile_variant(int N);
// xmode (coarse-to-fine initial guess, NEXT-4): 0 none; 1 write the final x of every system to xio (coarse half;
// carries x, i.e. the VERIFY arithmetic); 2 start from the P1 interpolation of the coarse solutions in xio.
cudaError_t launch_minres_tile(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                               unsigned* ctr, bool verify, const int* order, cudaStream_t s, int xmode = 0,
                               double* xio = nullptr);
// K3 for N >= 128: vectors in a per-CTA global scratch (nctas CTAs, minres_gm_scratch_per_cta(N) bytes each).
constexpr int kGmMinN = 128;
size_t minres_gm_scratch_per_cta(int N);
cudaError_t launch_minres_gm(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                             unsigned* job_counter, double* scratch, int nctas, cudaStream_t s);
// K3c for N = 128, 256, 512: one pass per MINRES step streamed through HBM with TMA-tiled planes
// (k_minres_stream.cu); same scratch convention (nctas CTAs x minres_stream_scratch_per_cta(N) bytes).
bool minres_stream_supported(int N);
// K3b: MINRES of one system per thread-block cluster, every row resident on chip (h = 1/128: 4 CTAs, 1/256: 16)
bool minres_cluster_supported(int N);
// job trace of the tile / K3b MINRES kernels (tuning build only; cudaErrorNotSupported otherwise)
cudaError_t minres_trace(unsigned long long* buf, unsigned cap, unsigned* count);
cudaError_t launch_minres_cluster(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                                  unsigned* ctr, const int* order, cudaStream_t s);
// Tiled TMA tensor map (cuTensorMapEncodeTiled via the runtime's driver entry point): `map` points to a
// CUtensorMap, dims innermost first, strides in bytes for dims 1.., zero OOB fill.  false on failure.
bool encode_tensor_map(void* map, bool f64, int rank, void* base, const uint64_t* dims, const uint64_t* strides,
                       const uint32_t* box);
size_t minres_stream_scratch_per_cta(int N);
cudaError_t launch_minres_stream(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                                 unsigned* job_counter, double* scratch, int nctas, cudaStream_t s,
                                 const int* order = nullptr);
int minres_stream_cluster(int N);   // CTAs per system of a streamed MINRES launch (a function of the mesh)
// K3m (NEXT-4): multigrid-preconditioned CG (k_mgcg.cu), same record convention.  N = 8..64 on chip;
// N = 128..512 one CTA per system over nctas x mgcg_scratch_per_cta(N) bytes of global scratch.
bool mgcg_supported(int N);
size_t mgcg_scratch_per_cta(int N);
int mgcg_ctas_per_sm(int N);   // resident systems per SM of the streamed-mesh MG-PCG
// nb_dev (optional, device): the number of systems, read by the kernel (escalation lists); ok_status: the
// status recorded for a converged solve (0; 4 = converged after escalation).
cudaError_t launch_mgcg(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                        unsigned* job_counter, const int* order, void* scratch, int nctas, cudaStream_t s,
                        const int* nb_dev = nullptr, int ok_status = 0);
// Plain CG (NEXT-4): the on-chip MG-PCG kernel without its preconditioner (z = r), N = 8 .. 64.
bool cg_supported(int N);
cudaError_t launch_cg(int N, const double* a, uint64_t nb, double tol, int max_iter, double* out, int slot,
                      unsigned* ctr, const int* order, cudaStream_t s);
// K4: banded Cholesky in u_f + Algorithm 1 refinement.  The factors go to a global scratch of
// chol_scratch_bytes(N, u_f, u_s, nb) bytes for a launch over nb systems (one factor per resident
// warp segment; a smaller scratch shrinks the grid; 0 = unsupported).
// u: the working precision u = u_r of x and the residual (MLMC_FMT_F64 default, MLMC_FMT_F32 or MLMC_FMT_F16).
cudaError_t launch_chol_ir(int N, const double* a, uint64_t nb, int u_f, int u_s, double tol, int i_max,
                           double* out, int slot, unsigned* job_counter, void* fscratch, size_t fbytes,
                           cudaStream_t s, int u = MLMC_FMT_F64);
bool chol_supported(int N, int u_f, int u_s, int u = MLMC_FMT_F64);
size_t chol_scratch_bytes(int N, int u_f, int u_s, uint64_t nb, int u = MLMC_FMT_F64);
// Escalation: the samples of `rec` whose slot-`slot` solve failed -> list[*count] (count zeroed by caller).
cudaError_t launch_escalate_collect(const double* rec, uint64_t nb, int slot, int* list, int* count, cudaStream_t s);
// K5: per-level sums of the per-sample records into sums (accumulate = add to existing).
// xsums (optional, device, kXLen words): the exact fixed-point sums, accumulated like sums.  chunk_scratch
// holds (kSumsLen + kXLen) x 8 bytes per chunk.
// Work model of one coupled sample's halves (R5): fixed + step x iterations; *_esc: an escalated half
// (status 4: failed attempt + MG-PCG re-solve, the record holding the MG-PCG steps).
struct CostParams {
    double f_fixed, f_step, f_esc, f_esc_step, c_fixed, c_step, c_esc, c_esc_step;
};
cudaError_t launch_level_sums(const double* rec, uint64_t nb, int level, const CostParams& cp, double* chunk_scratch,
                              double* sums, bool accumulate, cudaStream_t s, unsigned long long* xsums = nullptr);
// The exact fixed-point sums of the levels of the last mlmc_sample_levels(_async) call (nlev x kXLen words)
int copy_xsums_to_host(mlmc_ctx* ctx, int nlev, unsigned long long* host);
void ctx_want_xsums(mlmc_ctx* ctx, bool on);
double* ctx_adaptive_sums(mlmc_ctx* ctx);      // persistent device buffer of mlmc_adaptive_run's round sums   // form the exact sums in the sampling calls that follow

// Copy nlev level-sum records from the device to the host on the ctx's stream and wait.
int copy_sums_to_host(mlmc_ctx* ctx, const double* dev, int nlev, double* host);
// policy 3 (auto): the choice made for mesh N in tolerance class cls and its pilot cost (device ms/sample)
void ctx_note_auto_choice(mlmc_ctx* ctx, int N, int cls, const mlmc_precision& p, double ms_per_sample);
bool ctx_find_auto_choice(const mlmc_ctx* ctx, int N, int cls, mlmc_precision* p);

// Launch limits of a kernel.  cudaFuncSetAttribute (MaxDynamicSharedMemorySize) is per DEVICE, so the
// limits are cached per device ordinal: each call site keeps a `static PerDevice<KernelOcc>` and asks it with
// the launching device current; the first call on a device runs the initialiser under std::call_once, so
// several host threads driving contexts on one or several GPUs never see a half-written entry
// (a process-wide static skipped the attribute on a second device).
struct KernelOcc {
    cudaError_t err = cudaSuccess;
    int per_sm = 0;   // resident blocks per SM
    int sms = 0;
};
constexpr int kMaxDevices = 64;
template <class T>
struct PerDevice {
    T val[kMaxDevices];
    std::once_flag once[kMaxDevices];
    // the entry of the current device, initialised by init() on first use; dev_err set if no device
    template <class Init>
    const T& get(Init&& init, cudaError_t* dev_err = nullptr) {
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess || dev < 0 || dev >= kMaxDevices) {
            if (dev_err) *dev_err = e != cudaSuccess ? e : cudaErrorInvalidDevice;
            dev = 0;
        }
        std::call_once(once[dev], [&] { val[dev] = init(); });
        return val[dev];
    }
};
template <class Kern>
KernelOcc kernel_occ(Kern kern, int block, size_t smem) {
    KernelOcc o;
    o.err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (o.err == cudaSuccess) o.err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o.per_sm, kern, block, smem);
    int dev = 0;
    if (o.err == cudaSuccess) o.err = cudaGetDevice(&dev);
    if (o.err == cudaSuccess) o.err = cudaDeviceGetAttribute(&o.sms, cudaDevAttrMultiProcessorCount, dev);
    if (o.err == cudaSuccess && o.per_sm < 1) o.err = cudaErrorInvalidConfiguration;
    return o;
}
// cached per device: `static PerDevice<KernelOcc> cache; const KernelOcc occ = occ_of(cache, kern, block, smem);`
template <class Kern>
KernelOcc occ_of(PerDevice<KernelOcc>& cache, Kern kern, int block, size_t smem) {
    cudaError_t de = cudaSuccess;
    KernelOcc o = cache.get([&] { return kernel_occ(kern, block, smem); }, &de);
    if (de != cudaSuccess) o.err = de;
    return o;
}

// K3d (k_dd.cu, NEXT-3): MINRES of one sample over row slabs; state of the scalar recurrences (device).
struct DDState {
    double tol, beta1, inv_beta1, tol_b, invb_prev, alpha_prev, sigma_prev, dbar, epsln, phibar, cs, sn, s1q, s2q,
        Xq, ct, c1, c0, Q, relres;
    int max_iter, k, step, status, done, pad;
};
int dd_tiles(int N, int j0, int j1);
cudaError_t launch_dd_init(const double* a, int N, int j0, int rows, int pitch, double* planes, size_t plane_stride,
                           DDState* st, double tol, int max_iter, cudaStream_t s);
cudaError_t launch_dd_pass(int N, int j0, int j1, int rows, int pitch, double* planes, size_t plane_stride,
                           DDState* st, double* partials, unsigned* counter, double* sums, bool fuse_scalar,
                           cudaStream_t s);
cudaError_t launch_dd_scalar(DDState* st, const double* sums, int N, cudaStream_t s);
// World > 1 with the exchange fused into the kernel over peer memory (dd_peer_kernel); ranks rank0 ..
// rank0 + nranks - 1 in this launch, every pointer of every rank device-accessible from the launching GPU.
constexpr int kDDMaxRanks = 8;
struct DDPeerLaunch {
    int N, world, rank0, nranks;
    int j0[kDDMaxRanks], j1[kDDMaxRanks], rows[kDDMaxRanks];
    double* planes[kDDMaxRanks];
    size_t plane_stride[kDDMaxRanks];
    DDState* st[kDDMaxRanks];
    double* partials[kDDMaxRanks];
    unsigned* counter[kDDMaxRanks];
    double* rpart[kDDMaxRanks];
    unsigned* xcounter[kDDMaxRanks];
    double* sums[kDDMaxRanks];
};
cudaError_t launch_dd_peer(const DDPeerLaunch& L, cudaStream_t s);
// world = 1: the whole solve in one cooperative launch (partials needs 6 x tiles doubles)
cudaError_t launch_dd_persistent(int N, int j0, int j1, int rows, int pitch, double* planes, size_t plane_stride,
                                 DDState* st, double* partials, unsigned* counter, double* sums, cudaStream_t s);

constexpr int kSumsLen = MLMC_SUMS_LEN;
// Reproducible level sums: the five real-valued sums (Y, Y^2, Q_f, Q_c, cost) are also kept as
// exact fixed-point integers -- each per-sample value rounded once to a multiple of 2^-kXScale, added as a
// 256-bit two's-complement integer (4 little-endian 64-bit limbs) plus a count of values outside
// |x| < 2^62 (NaN, inf, huge; the double sums are used then).  Integer addition is associative, so the
// totals do not depend on how the samples were split over passes, chunks or ranks.
constexpr int kXFields = 5, kXWords = 5, kXLen = kXFields * kXWords, kXScale = 192;
constexpr int kRecLen = MLMC_SAMPLE_LEN;
constexpr uint64_t kChunk = 4096;

}  // namespace mlmc
