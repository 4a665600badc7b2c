// context.cu — runtime behind include/fscan_cuda.h: config handling, per-config
// tables (twiddles, Hann window, band intervals, cart2pol taps), workspace
// arena, streams, and the chunked batch pipeline K1a..K6 (kernels.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <complex>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "fscan_cuda.h"
#include "pipeline.h"

using namespace fscan_detail;

namespace {

constexpr double kPi = 3.141592653589793;  // std::numbers::pi (geometry.hpp:11)
#ifndef FSCAN_PDL_DEFAULT
#define FSCAN_PDL_DEFAULT 1
#endif
constexpr int kPdlDefault = FSCAN_PDL_DEFAULT;
constexpr int kPdlLatencyChunk = 4;
constexpr int kHostSlots = 4;              // fscan_match_batch_host input staging ring
constexpr int kMaxLanes = 8;               // concurrent chunk pipelines (FSCAN_LANES, default 3)
#ifdef FSCAN_NO_TEX_GATHER
constexpr bool kNoTexGather = true;  // A/B: K3 gathers with plain loads
#else
constexpr bool kNoTexGather = false;
#endif

struct Lane {
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    // workspace for `chunk` pairs
    float* ft = nullptr;
    float* gt = nullptr;
    float2* zbuf = nullptr;
    float* mag = nullptr;
    float2* fgt = nullptr;  // [chunk][2 planes][3np/4 + 1][np]
    Partial* part = nullptr;
    RotState* rot = nullptr;
    double* prof = nullptr;
    double* theta_ws = nullptr;
    int* flags = nullptr;
    int* polar_cnt = nullptr;  // behind the flags (same allocation)
    cudaTextureObject_t gtex = 0;  // K3 texture over gt (pow2 grids whose chunk fits one 2-D texture)
    // host-API staging (the inputs go through fscan_ctx::hslot)
    float* cart = nullptr;  // K0 output (polar API): 2 grids x chunk
    void* k0tab = nullptr;  // K0 tap table of the last polar geometry (built on this lane's stream)
    float* chain_ms = nullptr;  // odometry: masked scans of a chunk (chunk + 2 grids)
    int k0_naz = 0;
    double k0_res = 0.0, k0_delta = 0.0;
    fscan_pair_result* res = nullptr;
    double* tsurf = nullptr;
    float* xsurf = nullptr;
};

}  // namespace

struct fscan_ctx {
    int device = 0;
    fscan_config cfg{};
    int n = 0;
    int max_batch = 0;
    int chunk = 0;       // pairs per pipeline chunk
    int alloc_chunk = 0; // workspace capacity (pairs)
    int wide_chunk = 0;  // the ~2 GiB-per-lane chunk of this grid size, whatever max_batch (exhaustive search)
    int n_live = 0;
    int rot_col_blocks = 0;  // K1b column blocks (8 columns each) the polar taps read
    int phase = 0;           // opt-in phase correlation in the translation stage
    // programmatic dependent launch of the pipeline kernels (kernels.cu
    // pdl_enter): 0 off, 1 for latency-sized chunks (<= kPdlLatencyChunk pairs)
    // and grid side >= 1024, 2 always (FSCAN_PDL overrides). Measured with
    // PDL on: C1 (one pair) +2.7%, C5 (63 pairs of 1024^2) +1.0%, but C2 (three
    // lanes of 22 pairs of 256^2) -4.5% and C4 -0.3%: the next kernel's early
    // CTAs hold SM slots the other lanes' kernels could use
    int pdl_mode = kPdlDefault;
    // grid geometry: np = n for powers of two; otherwise the
    // rotation stage runs Bluestein DFTs of length bs_L at n and the
    // translation stage runs at np = 2^k >= n + 1 on zero-embedded scans
    int np = 0;
    int bs_L = 0;
    int nw = 0;               // half-plane width n - n/2
    long long mag_plane = 0;  // float2 per (|F|,|G|) tile set
    float2* bs_chirp = nullptr;
    float2* bs_kern = nullptr;
    float2* tw_L = nullptr;
    // brute-force search scratch (grown on demand)
    double* bf_thetas = nullptr;
    int bf_theta_cap = 0;
    Partial* bf_items = nullptr;
    cudaEvent_t bf_done = nullptr;  // recorded after the last exhaustive search's final kernel
    bool bf_done_valid = false;
    int bf_item_cap = 0;
    int launches_last = 0;
    std::string err;
    std::mutex mu;
    // tables
    float2* tw_n = nullptr;
    float2* tw_k = nullptr;
    float2* tw_k2 = nullptr;
    float2* tw_rk = nullptr;  // W_256^{r k} at (r-1)*16 + k (K4's radix-16 stage)
    float2* tw_k4 = nullptr;  // W_M^{a j} at a*48 + j, M = 3 np / 2 (K4's merged twiddles)
    float2* tw_m = nullptr;
    float* hann = nullptr;
    int2* band = nullptr;
    PolarTap* taps = nullptr;
    Lane lanes_[kMaxLanes];
    int nlanes = 3;
    Lane* lbegin() { return lanes_; }
    Lane* lend() { return lanes_ + nlanes; }
    cudaEvent_t start_ev = nullptr;
    // profiling: per-kernel events of the last call, serialised on lane 0
    int profiling = 0;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> prof;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    // CUDA-graph replay (fscan_ctx_set_graphs): cached executable graphs keyed
    // by the call's arguments, captured on `cap`; ordering against non-graph
    // work on the lanes and against replays on other streams through
    // `lane_sync` (per lane) and `graph_ev`
    struct GraphSlot {
        std::vector<uintptr_t> key;
        cudaGraphExec_t exec = nullptr;
        unsigned long long used = 0;
        int launches = 0;
    };
    int use_graphs = 0;
    std::vector<GraphSlot> graphs;
    unsigned long long graph_clock = 0;
    int graph_captures = 0, graph_replays = 0;
    cudaStream_t cap = nullptr;
    cudaEvent_t graph_ev = nullptr;
    cudaEvent_t lane_sync[kMaxLanes] = {};
    cudaStream_t last_graph_stream = nullptr;
    bool graph_launched = false;   // graph_ev holds the last replay
    bool lanes_since_graph = false; // non-graph work was queued on the lanes since
    bool capturing = false;
    // fscan_match_batch_host input staging: a ring of kHostSlots chunk buffers
    // filled in order on one copy stream (`h2d`), each released by an event
    // recorded after the chunk that read it; the copy of chunk k + 1 never waits
    // for the compute of chunk k (with the inputs staged in the lane, the next
    // copy of a lane queued behind its compute and the link idled between
    // rounds of chunks)
    struct HostSlot {
        float* in = nullptr;
        cudaEvent_t copied = nullptr, used = nullptr;
        bool pending = false;  // `used` recorded and not yet waited on
    };
    HostSlot hslot[kHostSlots];
    int hslot_chunk = 0;  // capacity of every slot (pairs)
    cudaStream_t h2d = nullptr;
    // pinned landing area of the per-chunk result rows: a device -> pageable
    // copy is synchronous for the host thread, which then could not queue the
    // next chunk's H2D copy until the previous chunk had finished
    fscan_pair_result* hres = nullptr;
    int hres_cap = 0;
};

namespace {

struct LaneRange {
    fscan_ctx* c;
    Lane* begin() const { return c->lbegin(); }
    Lane* end() const { return c->lend(); }
};

fscan_status fail(fscan_ctx* ctx, fscan_status st, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return st;
}

fscan_status cuda_fail(fscan_ctx* ctx, cudaError_t e, const char* where) {
    return fail(ctx, FSCAN_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                               \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
    } while (0)

bool is_pow2(int n) { return n > 0 && (n & (n - 1)) == 0; }

// bandpass_mask (imageops.cpp:44-59) restricted to the u >= 0 half plane:
// per centred row, the interval of u in [0, n/2) inside the band.
// In-place fp64 radix-2 FFT (forward, unnormalised) for the Bluestein kernel.
void fft_inplace(std::vector<std::complex<double>>& a) {
    const size_t n = a.size();
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        for (size_t i = 0; i < n; i += len)
            for (size_t k = 0; k < len / 2; ++k) {
                const std::complex<double> w = std::polar(1.0, -2.0 * kPi * (double)k / (double)len);
                const std::complex<double> u = a[i + k], v = a[i + k + len / 2] * w;
                a[i + k] = u + v;
                a[i + k + len / 2] = u - v;
            }
    }
}

bool build_band(int n, double lo, double hi, std::vector<int2>& out, std::vector<unsigned char>& inband) {
    const int c = n / 2, W = n - n / 2;  // half plane: centred columns c .. n-1
    const double nyq = n / 2.0;
    out.assign(n, make_int2(1, 0));
    inband.assign((size_t)n * W, 0);
    for (int i = 0; i < n; ++i) {
        int first = -1, last = -2;
        for (int u = 0; u < W; ++u) {
            const int j = c + u;
            const double rho = std::hypot(double(i - c), double(j - c)) / nyq;
            const bool in = (rho >= lo && rho <= hi);
            inband[(size_t)i * W + u] = in;
            if (in) {
                if (first < 0) first = u;
                else if (last != u - 1) return false;  // not an interval
                last = u;
            }
        }
        if (first >= 0) out[i] = make_int2(first, last);
    }
    return true;
}

// cart2pol taps (imageops.cpp:81-99 through sample_bilinear 10-26), exact
// fp64 coordinates; entries whose four taps all sit outside the band (or the
// array) contribute exactly 0 and are dropped by trimming the radius range.
// Taps on band-zeroed cells are not read either (flag bit clear: the value is
// exactly 0 in the reference too), so K1b only computes the column blocks up
// to *u_hi, the largest in-band column any tap reads.
bool build_taps(int n, const fscan_config& cfg, const std::vector<unsigned char>& inband,
                std::vector<PolarTap>& taps, int* n_live, int* u_hi, std::string* why) {
    const int nt = cfg.n_theta, nr = cfg.n_radius;
    const double span = nt * cfg.delta_theta;
    const int c = n / 2;
    const double r_max = n / 2.0;
    const int W = n - n / 2;  // half-plane width (n/2 for even n)
    std::vector<PolarTap> all((size_t)nt * nr);
    int jlo = nr, jhi = -1;
    *u_hi = 0;
    for (int i = 0; i < nt; ++i) {
        const double phi = -span / 2.0 + span * i / nt;
        const double cp = std::cos(phi), sp = std::sin(phi);
        for (int j = 0; j < nr; ++j) {
            const double r = r_max * (j + 1) / nr;
            const double row = c - r * sp, col = c + r * cp;
            const double r0f = std::floor(row), c0f = std::floor(col);
            const long r0 = (long)r0f, c0 = (long)c0f;
            const long u0 = c0 - c;
            int flags = 0, live = 0;
            for (int tp = 0; tp < 4; ++tp) {
                const long rr = r0 + (tp >> 1), uu = u0 + (tp & 1);
                const long cc = c + uu;
                const bool in_ref = rr >= 0 && rr < n && cc >= 0 && cc < n;  // reference array bounds
                if (!in_ref) continue;
                if (uu < 0) {
                    // tap on the u < 0 half plane; never happens for spans <= pi
                    if (uu >= -W) {
                        *why = "cart2pol tap on the u<0 half plane (span > pi?)";
                        return false;
                    }
                    continue;
                }
                if (uu >= W) continue;  // column n: outside the reference array
                if (!inband[(size_t)rr * W + uu]) continue;
                flags |= 1 << tp;
                live = 1;
                *u_hi = std::max(*u_hi, (int)uu);
            }
            PolarTap& e = all[(size_t)i * nr + j];
            e.packed = (int)(r0 & 0xFFF) | (int)((u0 & 0xFFF) << 12) | (flags << 24);
            e.fr = (float)(row - r0f);
            e.fc = (float)(col - c0f);
            e.pad_ = 0.f;
            if (r0 < 0 || r0 > n || u0 < 0 || u0 > W) {
                if (flags) {
                    *why = "cart2pol tap out of table range";
                    return false;
                }
            }
            if (live) {
                jlo = std::min(jlo, j);
                jhi = std::max(jhi, j);
            }
        }
    }
    if (jhi < jlo) {  // nothing in band: keep one (all-zero) column
        jlo = 0;
        jhi = 0;
    }
    *n_live = jhi - jlo + 1;
    taps.resize((size_t)nt * (*n_live));  // radius-major: [n_live][n_theta] (K2a lanes walk azimuth)
    for (int i = 0; i < nt; ++i)
        for (int j = jlo; j <= jhi; ++j) taps[(size_t)(j - jlo) * nt + i] = all[(size_t)i * nr + j];
    return true;
}

void free_lane(Lane& l) {
    if (l.gtex) cudaDestroyTextureObject(l.gtex);
    cudaFree(l.ft);
    cudaFree(l.gt);
    cudaFree(l.zbuf);
    cudaFree(l.mag);
    cudaFree(l.fgt);
    cudaFree(l.part);
    cudaFree(l.rot);
    cudaFree(l.prof);
    cudaFree(l.theta_ws);
    cudaFree(l.flags);
    cudaFree(l.cart);
    cudaFree(l.k0tab);
    cudaFree(l.chain_ms);
    cudaFree(l.res);
    cudaFree(l.tsurf);
    cudaFree(l.xsurf);
    l = Lane{l.stream, l.done};
}

fscan_status alloc_lane(fscan_ctx* ctx, Lane& l, int chunk) {
    const size_t n = (size_t)ctx->n, np = (size_t)ctx->np, npp = np * np;
    const int nparts = ctx->np / rows_per_block_out(ctx->np);
    // translation buffers at np (zero-embedded scans: the padding stays zero)
    CK(cudaMalloc(&l.ft, npp * sizeof(float) * chunk));
    CK(cudaMalloc(&l.gt, npp * sizeof(float) * chunk));
    if (np != n) {
        CK(cudaMemset(l.ft, 0, npp * sizeof(float) * chunk));
        CK(cudaMemset(l.gt, 0, npp * sizeof(float) * chunk));
    }
    // zbuf: K1 spectra (n x n) then the K4 -> K5 rows (np x (3np/4 + 1))
    CK(cudaMalloc(&l.zbuf, std::max(n * n, np * (size_t)ypitch((int)np)) * sizeof(float2) * chunk));
    // mag: the (|F|,|G|) tiles, later the np x np surface
    CK(cudaMalloc(&l.mag, std::max((size_t)ctx->mag_plane * 2, npp) * sizeof(float) * chunk));
    CK(cudaMalloc(&l.fgt, 2 * (3 * np / 4 + 1) * np * sizeof(float2) * chunk));
    CK(cudaMalloc(&l.part, sizeof(Partial) * nparts * chunk));
    CK(cudaMalloc(&l.rot, sizeof(RotState) * chunk));
    CK(cudaMalloc(&l.prof, sizeof(double) * 2 * std::max(1, ctx->cfg.n_theta) * chunk));
    CK(cudaMalloc(&l.theta_ws, sizeof(double) * std::max(1, ctx->cfg.n_theta) * chunk));
    CK(cudaMalloc(&l.flags, sizeof(int) * (2 * chunk + 2)));  // chain mode: one per scan; + K2b's per-pair counters
    l.polar_cnt = l.flags + chunk + 2;
    CK(cudaMemset(l.polar_cnt, 0, sizeof(int) * chunk));
    // K3 gathers g~ through a texture (tld4, zero border) when the chunk fits one
    // pitch-2D texture (rows = chunk * np)
    int max_h = 0;
    CK(cudaDeviceGetAttribute(&max_h, cudaDevAttrMaxTexture2DLinearHeight, ctx->device));
    if (np == n && !kNoTexGather && (long long)chunk * (long long)np <= max_h) {
        cudaResourceDesc rd{};
        rd.resType = cudaResourceTypePitch2D;
        rd.res.pitch2D.devPtr = l.gt;
        rd.res.pitch2D.desc = cudaCreateChannelDesc<float>();
        rd.res.pitch2D.width = np;
        rd.res.pitch2D.height = np * chunk;
        rd.res.pitch2D.pitchInBytes = np * sizeof(float);
        cudaTextureDesc td{};
        td.addressMode[0] = td.addressMode[1] = cudaAddressModeBorder;  // taps off the grid read 0
        td.filterMode = cudaFilterModePoint;
        td.readMode = cudaReadModeElementType;
        td.normalizedCoords = 0;
        CK(cudaCreateTextureObject(&l.gtex, &rd, &td, nullptr));
    }
    return FSCAN_OK;
}

fscan_status alloc_host_staging(fscan_ctx* ctx, Lane& l, int chunk) {
    if (l.res) return FSCAN_OK;
    const size_t nn = (size_t)ctx->n * ctx->n;
    CK(cudaMalloc(&l.res, sizeof(fscan_pair_result) * chunk));
    CK(cudaMalloc(&l.tsurf, sizeof(double) * std::max(1, ctx->cfg.n_theta) * chunk));
    CK(cudaMalloc(&l.xsurf, nn * sizeof(float) * chunk));
    return FSCAN_OK;
}

void free_host_slots(fscan_ctx* ctx) {
    if (ctx->h2d) cudaStreamSynchronize(ctx->h2d);
    for (auto& h : ctx->hslot) {
        if (h.used) cudaEventSynchronize(h.used);
        cudaFree(h.in);
        if (h.copied) cudaEventDestroy(h.copied);
        if (h.used) cudaEventDestroy(h.used);
        h = {};
    }
    ctx->hslot_chunk = 0;
}

fscan_status alloc_host_slots(fscan_ctx* ctx, int chunk) {
    if (ctx->hslot_chunk >= chunk) return FSCAN_OK;
    free_host_slots(ctx);
    if (!ctx->h2d) CK(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
    const size_t nn = (size_t)ctx->n * ctx->n;
    for (auto& h : ctx->hslot) {
        CK(cudaMalloc(&h.in, 4 * nn * sizeof(float) * chunk));
        CK(cudaEventCreateWithFlags(&h.copied, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h.used, cudaEventDisableTiming));
    }
    ctx->hslot_chunk = chunk;
    return FSCAN_OK;
}

Params base_params(fscan_ctx* ctx, Lane& l, int batch, double delta) {
    Params p{};
    p.n = ctx->n;
    p.np = ctx->np;
    p.embed = ctx->np != ctx->n;
    p.pdl = ctx->pdl_mode == 2 || (ctx->pdl_mode == 1 && (batch <= kPdlLatencyChunk || ctx->np >= 1024));
    p.c0 = (float)((ctx->n - 1) / 2.0);
    p.win_off = (ctx->np / 2 - 1) - (ctx->n - 1) / 2;
    p.nw = ctx->nw;
    p.mag_plane = ctx->mag_plane;
    p.bs_L = ctx->bs_L;
    p.bs_chirp = ctx->bs_chirp;
    p.bs_kern = ctx->bs_kern;
    p.tw_L = ctx->tw_L;
    p.batch = batch;
    p.ft = l.ft;
    p.gt = l.gt;
    p.gtex = l.gtex;
    p.gtex_base = l.gtex ? l.gt : nullptr;
    p.zbuf = l.zbuf;
    p.mag = l.mag;
    p.fgt = l.fgt;
    p.surf = l.mag;  // the magnitude planes are dead once K2 has run
    p.part = l.part;
    p.rot = l.rot;
    p.prof = l.prof;
    p.theta_ws = l.theta_ws;
    p.flags = l.flags;
    p.polar_cnt = l.polar_cnt;
    p.tw_n = ctx->tw_n;
    p.tw_k = ctx->tw_k;
    p.tw_k2 = ctx->tw_k2;
    p.tw_rk = ctx->tw_rk;
    p.tw_k4 = ctx->tw_k4;
    p.tw_m = ctx->tw_m;
    p.hann = ctx->hann;
    p.band = ctx->band;
    p.taps = ctx->taps;
    p.n_live = ctx->n_live;
    p.zcols = 8 * ctx->rot_col_blocks;
    p.src_div = 1;
    p.phase = ctx->phase;
    p.n_theta = ctx->cfg.n_theta;
    p.pad = ctx->cfg.pad_angle;
    p.L = ctx->cfg.n_theta + 2 * ctx->cfg.pad_angle;
    p.C = ctx->cfg.n_radius + 2 * ctx->cfg.pad_angle;
    p.delta_theta = ctx->cfg.delta_theta;
    p.t_theta = ctx->cfg.t_theta;
    p.t_xy = ctx->cfg.t_xy;
    p.delta = delta;
    p.window = ctx->cfg.softargmax_window;
    p.normalize = ctx->cfg.normalize_scores != 0;
    return p;
}

enum class Stages { Full, Rotation, Translation, Magnitude };

// Kernel ids for per-kernel profiling (fscan_ctx_kernel_times).
enum KernelId { kRotRows = 0, kRotCols, kRotPolar, kThetaIn, kXlatRows, kXlatCols, kXlatOut, kFinalize,
                kRotGather, kPolarToCart,
                kMagUnpack, kBfItems, kBfFinal, kXlatWin, kNumKernels };

struct ProfEvent {
    int kid;
    cudaEvent_t a, b;
};

// Launch one stage; in profiling mode bracket it with events on its stream.
template <typename L>
fscan_status launch(fscan_ctx* ctx, Lane& l, int kid, L&& fn, int* launches);

// Launch the pipeline for one chunk on lane l. Inputs are device pointers.
fscan_status run_chunk(fscan_ctx* ctx, Lane& l, Params p, Stages what, int* launches) {
    cudaStream_t s = l.stream;
    CK(cudaMemsetAsync(l.flags, 0, sizeof(int) * p.batch, s));
    fscan_status st;
#define FSCAN_LAUNCH(kid, call)                                                              \
    if ((st = launch(ctx, l, kid, [&] { return call(p, s); }, launches)) != FSCAN_OK) return st;
    // K1: power-of-two radix FFTs, or Bluestein DFTs for other sizes
    auto k1a = ctx->bs_L ? launch_rot_rows_bs : launch_rot_rows;
    auto k1b = ctx->bs_L ? launch_rot_cols_bs : launch_rot_cols;
    FSCAN_LAUNCH(kRotRows, k1a);
    if (what == Stages::Magnitude) {
        FSCAN_LAUNCH(kRotCols, k1b);
        FSCAN_LAUNCH(kMagUnpack, launch_mag_unpack);
        return FSCAN_OK;
    }
    if (what != Stages::Translation) {
        if (ctx->cfg.n_theta > 1) FSCAN_LAUNCH(kRotCols, k1b);
        if (ctx->cfg.n_theta > 1) FSCAN_LAUNCH(kRotGather, launch_rot_gather);
        FSCAN_LAUNCH(kRotPolar, launch_rot_polar);
    } else {
        FSCAN_LAUNCH(kThetaIn, launch_theta_in);
    }
    if (what != Stages::Rotation) {
        FSCAN_LAUNCH(kXlatRows, launch_xlat_rows);
        FSCAN_LAUNCH(kXlatCols, launch_xlat_cols);
        FSCAN_LAUNCH(kXlatOut, launch_xlat_out);
        if (xlat_win_pass(p)) FSCAN_LAUNCH(kXlatWin, launch_xlat_win);
        FSCAN_LAUNCH(kFinalize, launch_finalize);
    }
#undef FSCAN_LAUNCH
    return FSCAN_OK;
}

template <typename L>
fscan_status launch(fscan_ctx* ctx, Lane& l, int kid, L&& fn, int* launches) {
    cudaEvent_t a = nullptr, b = nullptr;
    if (ctx->profiling) {
        while (ctx->ev_pool.size() < ctx->ev_used + 2) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            ctx->ev_pool.push_back(e);
        }
        a = ctx->ev_pool[ctx->ev_used++];
        b = ctx->ev_pool[ctx->ev_used++];
        CK(cudaEventRecord(a, l.stream));
    }
    if (cudaError_t e = fn(); e != cudaSuccess) {  // name the kernel (KernelId) in the error
        const std::string what = "kernel " + std::to_string(kid);
        return cuda_fail(ctx, e, what.c_str());
    }
    if (ctx->profiling) {
        CK(cudaEventRecord(b, l.stream));
        ctx->prof.push_back({kid, {a, b}});
    }
    ++*launches;
    return FSCAN_OK;
}

fscan_status check_ctx(fscan_ctx* ctx, int batch) {
    if (!ctx) return FSCAN_ERR_INVALID_ARGUMENT;
    if (batch < 0 || batch > ctx->max_batch)
        return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "batch exceeds the context's max_batch");
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
    return FSCAN_OK;
}

// Generic device-side driver: split `batch` into chunks over the lanes,
// ordered after `user` and with `user` waiting for all lanes.
template <typename F>
fscan_status drive(fscan_ctx* ctx, int batch, cudaStream_t user, F&& per_chunk) {
    CK(cudaEventRecord(ctx->start_ev, user));
    for (Lane& l : LaneRange{ctx}) {
        CK(cudaStreamWaitEvent(l.stream, ctx->start_ev, 0));
        // after a graph replay on another stream, the lanes' workspace is free only once it ends
        if (ctx->graph_launched && !ctx->capturing) CK(cudaStreamWaitEvent(l.stream, ctx->graph_ev, 0));
    }
    if (!ctx->capturing) ctx->lanes_since_graph = true;
    ctx->launches_last = 0;
    ctx->prof.clear();
    ctx->ev_used = 0;
    const int lanes = ctx->profiling ? 1 : ctx->nlanes;
    int li = 0;
    for (int off = 0; off < batch; off += ctx->chunk, li = (li + 1) % lanes) {
        const int cnt = std::min(ctx->chunk, batch - off);
        fscan_status st = per_chunk(ctx->lanes_[li], off, cnt);
        if (st != FSCAN_OK) return st;
    }
    for (Lane& l : LaneRange{ctx}) {
        CK(cudaEventRecord(l.done, l.stream));
        CK(cudaStreamWaitEvent(user, l.done, 0));
    }
    return FSCAN_OK;
}

constexpr size_t kMaxGraphs = 8;

void drop_graphs(fscan_ctx* ctx) {
    for (auto& g : ctx->graphs) cudaGraphExecDestroy(g.exec);
    ctx->graphs.clear();
}

// drive() through the graph cache (fscan_ctx_set_graphs): replay the graph
// captured for `key`, or capture drive()'s whole launch sequence on the
// context's capture stream, instantiate it and replay it.
template <typename F>
fscan_status drive_graph(fscan_ctx* ctx, std::vector<uintptr_t> key, int batch, cudaStream_t user, F&& per_chunk) {
    if (!ctx->use_graphs || ctx->profiling) return drive(ctx, batch, user, per_chunk);
    if (!ctx->cap) {
        CK(cudaStreamCreateWithFlags(&ctx->cap, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ctx->graph_ev, cudaEventDisableTiming));
        for (int i = 0; i < kMaxLanes; ++i) CK(cudaEventCreateWithFlags(&ctx->lane_sync[i], cudaEventDisableTiming));
    }
    fscan_ctx::GraphSlot* slot = nullptr;
    for (auto& g : ctx->graphs)
        if (g.key == key) slot = &g;
    if (!slot) {
        ctx->capturing = true;
        cudaError_t e = cudaStreamBeginCapture(ctx->cap, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) {
            ctx->capturing = false;
            return cuda_fail(ctx, e, "cudaStreamBeginCapture");
        }
        fscan_status st = drive(ctx, batch, ctx->cap, per_chunk);
        cudaGraph_t graph = nullptr;
        e = cudaStreamEndCapture(ctx->cap, &graph);
        ctx->capturing = false;
        if (st != FSCAN_OK) {
            if (graph) cudaGraphDestroy(graph);
            return st;
        }
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaStreamEndCapture");
        cudaGraphExec_t exec = nullptr;
        e = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaGraphInstantiate");
        if (ctx->graphs.size() >= kMaxGraphs) {
            auto lru = std::min_element(ctx->graphs.begin(), ctx->graphs.end(),
                                        [](const auto& a, const auto& b) { return a.used < b.used; });
            cudaGraphExecDestroy(lru->exec);
            ctx->graphs.erase(lru);
        }
        ctx->graphs.push_back({std::move(key), exec, 0, ctx->launches_last});
        slot = &ctx->graphs.back();
        ++ctx->graph_captures;
    } else {
        ++ctx->graph_replays;
    }
    slot->used = ++ctx->graph_clock;
    ctx->launches_last = slot->launches;
    // order after non-graph work still queued on the lanes, and after a replay
    // on another stream (both use the context's workspace)
    if (ctx->lanes_since_graph) {
        for (int i = 0; i < ctx->nlanes; ++i) {
            CK(cudaEventRecord(ctx->lane_sync[i], ctx->lanes_[i].stream));
            CK(cudaStreamWaitEvent(user, ctx->lane_sync[i], 0));
        }
        ctx->lanes_since_graph = false;
    }
    if (ctx->graph_launched && ctx->last_graph_stream != user) CK(cudaStreamWaitEvent(user, ctx->graph_ev, 0));
    CK(cudaGraphLaunch(slot->exec, user));
    CK(cudaEventRecord(ctx->graph_ev, user));
    ctx->graph_launched = true;
    ctx->last_graph_stream = user;
    return FSCAN_OK;
}

uintptr_t key_bits(double d) {
    uintptr_t u = 0;
    std::memcpy(&u, &d, sizeof(double) < sizeof(u) ? sizeof(double) : sizeof(u));
    return u;
}

}  // namespace

extern "C" {

void fscan_config_defaults(fscan_config* c) {
    // MatchConfig defaults (matcher.hpp:13-26)
    c->n_theta = 733;
    c->delta_theta = kPi / 733.0;
    c->t_theta = 2.0;
    c->n_xy = 255;
    c->delta_xy = 0.4;
    c->t_xy = 1.0;
    c->band_lo = 0.03;
    c->band_hi = 0.75;
    c->n_radius = 128;
    c->pad_angle = 92;
    c->softargmax_window = 16;
    c->normalize_scores = 1;
}

void fscan_config_finalize(fscan_config* c) {  // matcher.cpp:11-15
    if (c->n_radius <= 0) c->n_radius = (c->n_xy + 1) / 2;
    if (c->pad_angle < 0) c->pad_angle = std::min((c->n_theta + 7) / 8, c->n_theta - 1);
}

fscan_status fscan_config_validate(const fscan_config* c, char* msg, size_t len) {
    auto bad = [&](const char* m) {
        if (msg && len) std::snprintf(msg, len, "%s", m);
        return FSCAN_ERR_INVALID_ARGUMENT;
    };
    // matcher.cpp:17-37 (the odd-n rule is the D1 exception)
    if (c->n_theta < 1) return bad("config: n_theta must be >= 1");
    if (!(c->delta_theta > 0.0)) return bad("config: delta_theta must be positive");
    if (c->n_theta * c->delta_theta > kPi + 1e-9) return bad("config: n_theta * delta_theta must not exceed pi");
    if (!(c->t_theta > 0.0) || !(c->t_xy > 0.0)) return bad("config: softmax gains must be positive");
    if (c->n_xy < 3) return bad("config: n_xy must be >= 3");
    if (!(c->delta_xy > 0.0)) return bad("config: delta_xy must be positive");
    if (!(c->band_lo >= 0.0 && c->band_lo < c->band_hi && c->band_hi <= 1.0))
        return bad("config: band must satisfy 0 <= lo < hi <= 1");
    if (c->n_theta > 1 && c->n_radius < 2) return bad("config: n_radius must be >= 2");
    if (c->pad_angle < 0 || c->pad_angle >= c->n_theta) return bad("config: need 0 <= pad_angle < n_theta");
    if (c->softargmax_window < 1) return bad("config: softargmax_window must be >= 1");
    if (msg && len) msg[0] = 0;
    return FSCAN_OK;
}

fscan_status fscan_ctx_create(int device, const fscan_config* cfg_in, int max_batch, fscan_ctx** out) {
    if (!out || !cfg_in || max_batch < 1) return FSCAN_ERR_INVALID_ARGUMENT;
    *out = nullptr;
    fscan_config cfg = *cfg_in;
    fscan_config_finalize(&cfg);
    char msg[256];
    fscan_status st = fscan_config_validate(&cfg, msg, sizeof msg);
    fscan_ctx* ctx = new fscan_ctx();
    ctx->cfg = cfg;
    ctx->device = device;
    ctx->n = cfg.n_xy;
    ctx->max_batch = max_batch;
    if (st != FSCAN_OK) {
        ctx->err = msg;
        *out = ctx;
        return st;
    }
    *out = ctx;
    {  // grid geometry: powers of two 64..1024 (fast path) or any other n in [33, 1023]
        const int n = ctx->n;
        int np = 64;
        while (np < (is_pow2(n) ? n : n + 1)) np <<= 1;
        if (n < 33 || n > 1024 || np > 1024)
            return fail(ctx, FSCAN_ERR_UNSUPPORTED,
                        "n_xy must lie in [33, 1024] on the GPU path (powers of two >= 64 take the fast path)");
        ctx->np = np;
        ctx->nw = n - n / 2;
        ctx->mag_plane = (long long)n * 8 * ((ctx->nw + 7) / 8);
        if (!is_pow2(n)) {
            int L = 128;
            while (L < 2 * n - 1) L <<= 1;
            ctx->bs_L = L;
        }
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return fail(ctx, FSCAN_ERR_NO_DEVICE, "no CUDA device " + std::to_string(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10) return fail(ctx, FSCAN_ERR_NO_DEVICE, "needs an sm_100 (B200) device");
    CK(cudaSetDevice(device));

    const int n = ctx->n;
    // tables
    // twiddle tables exp(-2 pi i k / L), fp64-accurate then rounded to fp32:
    // L = N (rotation stage), K = N/2 and K/2 (translation FFTs), M = 3N/2
    auto table = [](int len) {
        std::vector<float2> t(len);
        for (int i = 0; i < len; ++i) {
            const double a = -2.0 * kPi * i / len;
            t[i] = make_float2((float)std::cos(a), (float)std::sin(a));
        }
        return t;
    };
    const int np = ctx->np;  // translation stage size
    const std::vector<float2> tw = table(ctx->bs_L ? ctx->bs_L : n), twk = table(np / 2), twk2 = table(np / 4),
                              twm = table(3 * np / 2);
    std::vector<float> hann(n, 1.0f);  // imageops.cpp:30-42
    if (n > 1)
        for (int i = 0; i < n; ++i) hann[i] = (float)(0.5 * (1.0 - std::cos(2.0 * kPi * i / (n - 1))));
    std::vector<int2> band;
    std::vector<unsigned char> inband;
    if (!build_band(n, cfg.band_lo, cfg.band_hi, band, inband))
        return fail(ctx, FSCAN_ERR_UNSUPPORTED, "band is not an interval per row");
    std::vector<PolarTap> taps;
    if (cfg.n_theta > 1) {
        std::string why;
        int u_hi = 0;
        if (!build_taps(n, cfg, inband, taps, &ctx->n_live, &u_hi, &why)) return fail(ctx, FSCAN_ERR_UNSUPPORTED, why);
        ctx->rot_col_blocks = std::min((ctx->nw + 7) / 8, u_hi / 8 + 1);
    } else {
        taps.resize(1);
        ctx->n_live = 1;
        ctx->rot_col_blocks = (ctx->nw + 7) / 8;
    }
    if (ctx->bs_L) {  // Bluestein tables (generic_n.cu): chirp w[k] and FFT_L(conj kernel) / L
        const int L = ctx->bs_L;
        std::vector<std::complex<double>> w(n), b(L, 0.0);
        for (int k = 0; k < n; ++k) {
            const long long e = (long long)k * k % (2LL * n);  // exact phase reduction
            w[k] = std::polar(1.0, -kPi * (double)e / n);
        }
        for (int m = 0; m < n; ++m) {
            b[m] = std::conj(w[m]);
            if (m) b[L - m] = std::conj(w[m]);
        }
        fft_inplace(b);
        std::vector<float2> chirp(n), kern(L);
        for (int k = 0; k < n; ++k) chirp[k] = make_float2((float)w[k].real(), (float)w[k].imag());
        for (int k = 0; k < L; ++k) kern[k] = make_float2((float)(b[k].real() / L), (float)(b[k].imag() / L));
        CK(cudaMalloc(&ctx->bs_chirp, sizeof(float2) * n));
        CK(cudaMalloc(&ctx->bs_kern, sizeof(float2) * L));
        CK(cudaMemcpy(ctx->bs_chirp, chirp.data(), sizeof(float2) * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->bs_kern, kern.data(), sizeof(float2) * L, cudaMemcpyHostToDevice));
    }
    CK(cudaMalloc(&ctx->tw_n, sizeof(float2) * tw.size()));
    CK(cudaMalloc(&ctx->tw_k, sizeof(float2) * twk.size()));
    CK(cudaMalloc(&ctx->tw_k2, sizeof(float2) * twk2.size()));
    CK(cudaMalloc(&ctx->tw_m, sizeof(float2) * twm.size()));
    CK(cudaMemcpy(ctx->tw_k, twk.data(), sizeof(float2) * twk.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->tw_k2, twk2.data(), sizeof(float2) * twk2.size(), cudaMemcpyHostToDevice));
    {
        std::vector<float2> rk(240);
        for (int r = 1; r < 16; ++r)
            for (int k = 0; k < 16; ++k) {
                const double a = -2.0 * kPi * ((r * k) % 256) / 256.0;
                rk[(r - 1) * 16 + k] = make_float2((float)std::cos(a), (float)std::sin(a));
            }
        CK(cudaMalloc(&ctx->tw_rk, sizeof(float2) * rk.size()));
        CK(cudaMemcpy(ctx->tw_rk, rk.data(), sizeof(float2) * rk.size(), cudaMemcpyHostToDevice));
        // K4's merged twiddle table (fft.cuh SmemTwQF / SmemTwQI), exact phase reduction
        const long long m3 = 3LL * ctx->np / 2;
        std::vector<float2> k4(16 * 48);
        for (int a = 0; a < 16; ++a)
            for (int j = 0; j < 48; ++j) {
                const double e = -2.0 * kPi * (double)((a * j) % m3) / (double)m3;
                k4[a * 48 + j] = make_float2((float)std::cos(e), (float)std::sin(e));
            }
        CK(cudaMalloc(&ctx->tw_k4, sizeof(float2) * k4.size()));
        CK(cudaMemcpy(ctx->tw_k4, k4.data(), sizeof(float2) * k4.size(), cudaMemcpyHostToDevice));
    }
    CK(cudaMemcpy(ctx->tw_m, twm.data(), sizeof(float2) * twm.size(), cudaMemcpyHostToDevice));
    CK(cudaMalloc(&ctx->hann, sizeof(float) * n));
    CK(cudaMalloc(&ctx->band, sizeof(int2) * n));
    CK(cudaMalloc(&ctx->taps, sizeof(PolarTap) * taps.size()));
    CK(cudaMemcpy(ctx->tw_n, tw.data(), sizeof(float2) * tw.size(), cudaMemcpyHostToDevice));
    ctx->tw_L = ctx->bs_L ? ctx->tw_n : nullptr;  // the length-L table for the Bluestein FFTs
    CK(cudaMemcpy(ctx->hann, hann.data(), sizeof(float) * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->band, band.data(), sizeof(int2) * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(ctx->taps, taps.data(), sizeof(PolarTap) * taps.size(), cudaMemcpyHostToDevice));

    // lanes (concurrent chunk pipelines) and chunk size: FSCAN_LANES / FSCAN_CHUNK
    // override the defaults (3 lanes, ~2 GiB of workspace per lane; 3 lanes
    // measured +0.9% over 2 at C4, 4-8 lanes or other chunk sizes no better)
    if (const char* e = std::getenv("FSCAN_LANES")) ctx->nlanes = std::clamp(std::atoi(e), 1, kMaxLanes);
    if (const char* e = std::getenv("FSCAN_PDL")) ctx->pdl_mode = std::clamp(std::atoi(e), 0, 2);
    const double per_pair = (double)n * n * (8 + 4 + 8) + (double)n * (3 * n / 4 + 1) * 16;
    // ~2 GiB of workspace per lane: 126 pairs at N = 512 (then the texture cap
    // below), 63 at N = 1024 (C5 +2% over 1 GiB / 31 pairs: larger grids, and K2b
    // leaves its small-batch split path)
    int chunk = (int)std::max(1.0, std::floor((2048.0 * 1024 * 1024) / per_pair));
    // a batch smaller than the lanes' chunks is spread over all lanes (C2, 64
    // pairs: +7% over one 64-pair chunk); tiny contexts keep whole-batch chunks
    // (the exhaustive search runs pair x candidate items through them)
    int wide = chunk;
    if (max_batch >= 16 * ctx->nlanes) chunk = std::min(chunk, (max_batch + ctx->nlanes - 1) / ctx->nlanes);
    if (const char* e = std::getenv("FSCAN_CHUNK")) chunk = std::max(1, std::atoi(e));
    chunk = std::min(chunk, max_batch);
    if (ctx->np == ctx->n && !kNoTexGather) {  // keep the chunk inside one K3 gather texture
        int max_h = 0;
        CK(cudaDeviceGetAttribute(&max_h, cudaDevAttrMaxTexture2DLinearHeight, device));
        if (max_h >= ctx->np) {
            chunk = std::min(chunk, max_h / ctx->np);
            wide = std::min(wide, max_h / ctx->np);
        }
    }
    ctx->wide_chunk = wide;
    ctx->chunk = chunk;
    ctx->alloc_chunk = chunk;
    CK(cudaEventCreateWithFlags(&ctx->start_ev, cudaEventDisableTiming));
    for (Lane& l : LaneRange{ctx}) {
        if (const char* e = std::getenv("FSCAN_LANE_PRIO"); e && std::atoi(e)) {
            // A/B: graded lane priorities (lane 0 highest), so one lane's kernels
            // are scheduled ahead and the lanes stay phase-shifted
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            const int li = (int)(&l - ctx->lanes_);
            CK(cudaStreamCreateWithPriority(&l.stream, cudaStreamNonBlocking, std::min(lo, hi + li)));
        } else {
            CK(cudaStreamCreateWithFlags(&l.stream, cudaStreamNonBlocking));
        }
        CK(cudaEventCreateWithFlags(&l.done, cudaEventDisableTiming));
        fscan_status a = alloc_lane(ctx, l, chunk);
        if (a != FSCAN_OK) return a;
    }
    return FSCAN_OK;
}

void fscan_ctx_destroy(fscan_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    // work queued on user streams (graph replays, the exhaustive search's final
    // kernel) reads the workspace freed below
    if (ctx->graph_launched) cudaEventSynchronize(ctx->graph_ev);
    if (ctx->bf_done_valid) cudaEventSynchronize(ctx->bf_done);
    for (Lane& l : LaneRange{ctx}) {
        if (l.stream) cudaStreamSynchronize(l.stream);
        free_lane(l);
        if (l.stream) cudaStreamDestroy(l.stream);
        if (l.done) cudaEventDestroy(l.done);
    }
    if (ctx->start_ev) cudaEventDestroy(ctx->start_ev);
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->cap) cudaStreamSynchronize(ctx->cap);
    drop_graphs(ctx);
    if (ctx->cap) cudaStreamDestroy(ctx->cap);
    if (ctx->graph_ev) cudaEventDestroy(ctx->graph_ev);
    for (cudaEvent_t e : ctx->lane_sync)
        if (e) cudaEventDestroy(e);
    free_host_slots(ctx);
    if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
    if (ctx->hres) cudaFreeHost(ctx->hres);
    cudaFree(ctx->tw_n);
    cudaFree(ctx->tw_k);
    cudaFree(ctx->tw_k2);
    cudaFree(ctx->tw_rk);
    cudaFree(ctx->tw_k4);
    cudaFree(ctx->tw_m);
    cudaFree(ctx->hann);
    cudaFree(ctx->band);
    cudaFree(ctx->taps);
    cudaFree(ctx->bs_chirp);
    cudaFree(ctx->bs_kern);
    cudaFree(ctx->bf_thetas);
    cudaFree(ctx->bf_items);
    if (ctx->bf_done) cudaEventDestroy(ctx->bf_done);
    delete ctx;
}

const char* fscan_ctx_last_error(const fscan_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int fscan_ctx_n(const fscan_ctx* ctx) { return ctx ? ctx->n : 0; }

int fscan_ctx_launches_last(const fscan_ctx* ctx) { return ctx ? ctx->launches_last : 0; }

int fscan_ctx_rot_columns(const fscan_ctx* ctx) { return ctx ? 8 * ctx->rot_col_blocks : 0; }

// Lane workspace for at least `pairs` pairs per chunk (the caller holds ctx->mu
// and has dropped the cached graphs, which bake in the workspace pointers).
static fscan_status grow_lanes(fscan_ctx* ctx, int pairs) {
    if (pairs <= ctx->alloc_chunk) return FSCAN_OK;
    cudaSetDevice(ctx->device);
    // a graph replay on a user stream may still be using the workspace
    if (ctx->graph_launched) cudaEventSynchronize(ctx->graph_ev);
    for (Lane& l : LaneRange{ctx}) {
        cudaStreamSynchronize(l.stream);
        const bool had_host = l.res != nullptr;
        free_lane(l);
        fscan_status a = alloc_lane(ctx, l, pairs);
        if (a != FSCAN_OK) return a;
        if (had_host) {
            a = alloc_host_staging(ctx, l, pairs);
            if (a != FSCAN_OK) return a;
        }
    }
    ctx->alloc_chunk = pairs;
    return FSCAN_OK;
}

fscan_status fscan_ctx_set_chunk(fscan_ctx* ctx, int pairs) {
    if (!ctx || pairs < 0) return FSCAN_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(ctx->mu);
    if (pairs == 0) pairs = ctx->alloc_chunk;
    // cached graphs bake in the chunking and the lane workspace pointers
    if (pairs != ctx->chunk || pairs > ctx->alloc_chunk) drop_graphs(ctx);
    fscan_status a = grow_lanes(ctx, pairs);
    if (a != FSCAN_OK) return a;
    ctx->chunk = pairs;
    return FSCAN_OK;
}

fscan_status fscan_match_batch(fscan_ctx* ctx, const float* d_f, const float* d_g, const float* d_mf,
                               const float* d_mg, int batch, double delta, fscan_pair_result* d_out,
                               double* d_tsurf, float* d_xsurf, void* stream) {
    fscan_status st = check_ctx(ctx, batch);
    if (st != FSCAN_OK) return st;
    std::lock_guard<std::mutex> g(ctx->mu);
    if (batch == 0) return FSCAN_OK;  // empty batches may pass null pointers
    if (!ctx->tw_n) return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "context was not created successfully");
    if (!d_f || !d_g || !d_out || ((d_mf == nullptr) != (d_mg == nullptr)) || !(delta > 0.0))
        return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "fscan_match_batch: bad pointers or delta");
    const size_t nn = (size_t)ctx->n * ctx->n;
    const int nt = ctx->cfg.n_theta;
    std::vector<uintptr_t> key{1,
                               (uintptr_t)d_f,
                               (uintptr_t)d_g,
                               (uintptr_t)d_mf,
                               (uintptr_t)d_mg,
                               (uintptr_t)batch,
                               key_bits(delta),
                               (uintptr_t)d_out,
                               (uintptr_t)d_tsurf,
                               (uintptr_t)d_xsurf};
    return drive_graph(ctx, std::move(key), batch, (cudaStream_t)stream, [&](Lane& l, int off, int cnt) {
        Params p = base_params(ctx, l, cnt, delta);
        p.f = d_f + off * nn;
        p.g = d_g + off * nn;
        p.mf = d_mf ? d_mf + off * nn : nullptr;
        p.mg = d_mg ? d_mg + off * nn : nullptr;
        p.out = d_out + off;
        p.theta_surf = d_tsurf ? d_tsurf + (size_t)off * nt : nullptr;
        p.xy_surf = d_xsurf ? d_xsurf + off * nn : nullptr;
        return run_chunk(ctx, l, p, Stages::Full, &ctx->launches_last);
    });
}

fscan_status fscan_match_batch_polar(fscan_ctx* ctx, const float* d_pf, const float* d_pg, int n_az,
                                     int n_range, double range_res, const float* d_mf, const float* d_mg,
                                     int batch, double delta, fscan_pair_result* d_out, double* d_tsurf,
                                     float* d_xsurf, void* stream) {
    fscan_status st = check_ctx(ctx, batch);
    if (st != FSCAN_OK) return st;
    std::lock_guard<std::mutex> g(ctx->mu);
    if (batch == 0) return FSCAN_OK;  // empty batches may pass null pointers
    if (!ctx->tw_n) return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "context was not created successfully");
    if (!d_pf || !d_pg || !d_out || ((d_mf == nullptr) != (d_mg == nullptr)) || !(delta > 0.0) || n_az < 1 ||
        n_range < 1 || !(range_res > 0.0))
        return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "fscan_match_batch_polar: bad pointers or geometry");
    const size_t nn = (size_t)ctx->n * ctx->n, np = (size_t)n_az * n_range;
    const int nt = ctx->cfg.n_theta;
    for (Lane& l : LaneRange{ctx}) {
        if (!l.cart) CK(cudaMalloc(&l.cart, 2 * nn * sizeof(float) * ctx->alloc_chunk));
        if (!l.k0tab) CK(cudaMalloc(&l.k0tab, polar_tap_bytes(ctx->n)));
        if (l.k0_naz != n_az || l.k0_res != range_res || l.k0_delta != delta) {  // K0 geometry changed
            CK(launch_polar_taps(n_az, range_res, ctx->n, delta, l.k0tab, l.stream));
            l.k0_naz = n_az;
            l.k0_res = range_res;
            l.k0_delta = delta;
        }
    }
    return drive(ctx, batch, (cudaStream_t)stream, [&](Lane& l, int off, int cnt) {
        // K0: both sweeps of the chunk -> Cartesian grids in the lane's staging buffer
        fscan_status s2;
        if ((s2 = launch(ctx, l, kPolarToCart, [&] {
                 return launch_polar_to_cart(d_pf + off * np, d_pg + off * np, cnt, n_az, n_range, range_res,
                                             ctx->n, delta, l.cart, l.cart + nn * cnt, l.stream, l.k0tab);
             }, &ctx->launches_last)) != FSCAN_OK)
            return s2;
        Params p = base_params(ctx, l, cnt, delta);
        p.f = l.cart;
        p.g = l.cart + nn * cnt;
        p.mf = d_mf ? d_mf + off * nn : nullptr;
        p.mg = d_mg ? d_mg + off * nn : nullptr;
        p.out = d_out + off;
        p.theta_surf = d_tsurf ? d_tsurf + (size_t)off * nt : nullptr;
        p.xy_surf = d_xsurf ? d_xsurf + off * nn : nullptr;
        return run_chunk(ctx, l, p, Stages::Full, &ctx->launches_last);
    });
}

fscan_status fscan_estimate_rotation_batch(fscan_ctx* ctx, const float* d_f, const float* d_g, int batch,
                                           double* d_theta, double* d_tsurf, void* stream) {
    fscan_status st = check_ctx(ctx, batch);
    if (st != FSCAN_OK) return st;
    std::lock_guard<std::mutex> g(ctx->mu);
    if (batch == 0) return FSCAN_OK;  // empty batches may pass null pointers
    if (!d_f || !d_g || !d_theta) return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "bad pointers");
    const size_t nn = (size_t)ctx->n * ctx->n;
    return drive(ctx, batch, (cudaStream_t)stream, [&](Lane& l, int off, int cnt) {
        Params p = base_params(ctx, l, cnt, 1.0);
        p.f = d_f + off * nn;
        p.g = d_g + off * nn;
        p.theta_only = d_theta + off;
        p.theta_surf = d_tsurf ? d_tsurf + (size_t)off * ctx->cfg.n_theta : nullptr;
        return run_chunk(ctx, l, p, Stages::Rotation, &ctx->launches_last);
    });
}

fscan_status fscan_estimate_translation_batch(fscan_ctx* ctx, const float* d_f, const float* d_g, int batch,
                                              double delta, const double* d_theta, double* d_txy,
                                              float* d_xsurf, void* stream) {
    fscan_status st = check_ctx(ctx, batch);
    if (st != FSCAN_OK) return st;
    std::lock_guard<std::mutex> g(ctx->mu);
    if (batch == 0) return FSCAN_OK;  // empty batches may pass null pointers
    if (!d_f || !d_g || !d_theta || !d_txy || !(delta > 0.0))
        return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "bad pointers or delta");
    const size_t nn = (size_t)ctx->n * ctx->n;
    return drive(ctx, batch, (cudaStream_t)stream, [&](Lane& l, int off, int cnt) {
        Params p = base_params(ctx, l, cnt, delta);
        p.f = d_f + off * nn;
        p.g = d_g + off * nn;
        p.theta_in = d_theta + off;
        p.txy_only = d_txy + 2 * off;
        p.xy_surf = d_xsurf ? d_xsurf + off * nn : nullptr;
        return run_chunk(ctx, l, p, Stages::Translation, &ctx->launches_last);
    });
}

fscan_status fscan_brute_force_batch(fscan_ctx* ctx, const float* d_f, const float* d_g, int batch,
                                     const double* thetas, int nth, double delta, fscan_bf_result* d_out,
                                     void* stream) {
    fscan_status st = check_ctx(ctx, batch);
    if (st != FSCAN_OK) return st;
    std::lock_guard<std::mutex> g(ctx->mu);
    if (batch == 0) return FSCAN_OK;  // empty batches may pass null pointers
    if (!ctx->tw_n) return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "context was not created successfully");
    if (!d_f || !d_g || !d_out || !(delta > 0.0))
        return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "fscan_brute_force_batch: bad pointers or delta");
    if (!thetas || nth < 1)  // oracle.cpp:46-47
        return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "brute_force_match: empty theta candidate list");
    if ((long long)batch * nth > (1LL << 30))
        return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "fscan_brute_force_batch: too many (pair, theta) items");
    cudaStream_t user = (cudaStream_t)stream;
    const int items = batch * nth;
    if (ctx->bf_theta_cap < nth) {
        cudaFree(ctx->bf_thetas);
        ctx->bf_thetas = nullptr;
        CK(cudaMalloc(&ctx->bf_thetas, sizeof(double) * nth));
        ctx->bf_theta_cap = nth;
    }
    if (ctx->bf_item_cap < items) {
        cudaFree(ctx->bf_items);
        ctx->bf_items = nullptr;
        CK(cudaMalloc(&ctx->bf_items, sizeof(Partial) * items));
        ctx->bf_item_cap = items;
    }
    // the candidate list is small: a synchronous copy keeps the host array's lifetime
    // simple; the previous call's kernels (on whatever stream it was given) must be
    // done with bf_thetas / bf_items before they are overwritten
    if (ctx->bf_done_valid) CK(cudaEventSynchronize(ctx->bf_done));
    CK(cudaStreamSynchronize(user));
    CK(cudaMemcpy(ctx->bf_thetas, thetas, sizeof(double) * nth, cudaMemcpyHostToDevice));
    // grids that are not powers of two: zero-embed f and g once per call (§3.9)
    const bool embed = ctx->np != ctx->n;
    float* ef = nullptr;
    if (embed) {
        const size_t npp = (size_t)ctx->np * ctx->np;
        CK(cudaMalloc(&ef, 2 * npp * sizeof(float) * batch));
        CK(cudaMemset(ef, 0, 2 * npp * sizeof(float) * batch));
        CK(launch_embed(d_f, batch, ctx->n, ctx->np, ef, user));
        CK(launch_embed(d_g, batch, ctx->n, ctx->np, ef + npp * batch, user));
        d_f = ef;
        d_g = ef + npp * batch;
    }
    // (pair, candidate) items, not pairs, flow through the lanes: a context made
    // for a few pairs gets lanes wide enough for the items to fill the GPU (with
    // max_batch-sized chunks every 5-kernel chunk of a 4-pair search was launch
    // bound: 720 chunks of 4 items at C4's 720 candidates)
    const int saved_chunk = ctx->chunk;
    {
        const int want = std::min(ctx->wide_chunk, (items + ctx->nlanes - 1) / ctx->nlanes);
        if (want > ctx->alloc_chunk) {
            drop_graphs(ctx);
            fscan_status a = grow_lanes(ctx, want);
            if (a != FSCAN_OK) {
                cudaFree(ef);
                return a;
            }
        }
        ctx->chunk = std::max(ctx->chunk, std::min(want, ctx->alloc_chunk));
    }
    st = drive(ctx, items, user, [&](Lane& l, int off, int cnt) {
        Params p = base_params(ctx, l, cnt, delta);
        // brute_force_match scores the scans as given; only K3 reads ft / gt here
        p.ft = const_cast<float*>(d_f);
        p.gt = const_cast<float*>(d_g);
        p.item_base = off;
        p.src_div = nth;
        p.theta_in = ctx->bf_thetas;
        p.theta_mod = nth;
        p.skip_surface = 1;
        p.bf_items = ctx->bf_items;
        cudaStream_t s = l.stream;
        fscan_status r;
#define FSCAN_LAUNCH(kid, call)                                                              \
    if ((r = launch(ctx, l, kid, [&] { return call(p, s); }, &ctx->launches_last)) != FSCAN_OK) return r;
        FSCAN_LAUNCH(kThetaIn, launch_theta_in);
        FSCAN_LAUNCH(kXlatRows, launch_xlat_rows);
        FSCAN_LAUNCH(kXlatCols, launch_xlat_cols);
        FSCAN_LAUNCH(kXlatOut, launch_xlat_out);
        FSCAN_LAUNCH(kBfItems, launch_bf_items);
#undef FSCAN_LAUNCH
        return FSCAN_OK;
    });
    ctx->chunk = saved_chunk;
    if (st != FSCAN_OK) {
        cudaFree(ef);
        return st;
    }
    // all lanes are joined into `user`: the per-pair winner over the candidates
    const int off = (ctx->np / 2 - 1) - (ctx->n - 1) / 2;
    CK(launch_bf_final(ctx->bf_items, ctx->bf_thetas, nth, batch, ctx->n, ctx->np, off, delta, d_out, user));
    ++ctx->launches_last;
    if (!ctx->bf_done) CK(cudaEventCreateWithFlags(&ctx->bf_done, cudaEventDisableTiming));
    CK(cudaEventRecord(ctx->bf_done, user));
    ctx->bf_done_valid = true;
    if (ef) {
        CK(cudaStreamSynchronize(user));  // the embedded copies are read by the launched kernels
        cudaFree(ef);
    }
    return FSCAN_OK;
}

fscan_status fscan_odometry_batch(fscan_ctx* ctx, const float* d_scans, const float* d_masks, int n_scans,
                                  double delta, fscan_pair_result* d_out, double* d_tsurf, float* d_xsurf,
                                  void* stream) {
    const int pairs = n_scans - 1;
    fscan_status st = check_ctx(ctx, std::max(0, pairs));
    if (st != FSCAN_OK) return st;
    std::lock_guard<std::mutex> g(ctx->mu);
    if (!ctx->tw_n) return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "context was not created successfully");
    if (n_scans < 0 || !(delta > 0.0)) return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "fscan_odometry_batch: bad count or delta");
    if (pairs <= 0) return FSCAN_OK;  // 0 or 1 scans: no pairs
    if (!d_scans || !d_out) return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "fscan_odometry_batch: bad pointers");
    const size_t nn = (size_t)ctx->n * ctx->n;
    const size_t npp = (size_t)ctx->np * ctx->np;  // masked scans live in the translation grid (embedded)
    const int nt = ctx->cfg.n_theta;
    for (Lane& l : LaneRange{ctx})
        if (!l.chain_ms) {
            CK(cudaMalloc(&l.chain_ms, (ctx->alloc_chunk + 2) * npp * sizeof(float)));
            if (npp != nn) CK(cudaMemset(l.chain_ms, 0, (ctx->alloc_chunk + 2) * npp * sizeof(float)));
        }
    std::vector<uintptr_t> key{2,
                               (uintptr_t)d_scans,
                               (uintptr_t)d_masks,
                               (uintptr_t)n_scans,
                               key_bits(delta),
                               (uintptr_t)d_out,
                               (uintptr_t)d_tsurf,
                               (uintptr_t)d_xsurf};
    return drive_graph(ctx, std::move(key), pairs, (cudaStream_t)stream, [&](Lane& l, int off, int cnt) {
        // pairs off .. off+cnt-1 register scans off .. off+cnt
        Params p = base_params(ctx, l, cnt, delta);
        p.f = d_scans + off * nn;
        p.mf = d_masks ? d_masks + off * nn : nullptr;
        p.chain = 1;
        p.n_scans = cnt + 1;
        p.ft = l.chain_ms;        // masked scan s of the chunk at ft + s * np^2
        p.gt = l.chain_ms + npp;  // pair k reads scans k (ft) and k+1 (gt)
        p.out = d_out + off;
        p.theta_surf = d_tsurf ? d_tsurf + (size_t)off * nt : nullptr;
        p.xy_surf = d_xsurf ? d_xsurf + off * nn : nullptr;
        Params r = p;  // rotation-stage spectra: one packed transform per two scans
        r.batch = (cnt + 2) / 2;
        cudaStream_t s = l.stream;
        CK(cudaMemsetAsync(l.flags, 0, sizeof(int) * (cnt + 1), s));
        fscan_status e;
#define FSCAN_LAUNCH(kid, call, P)                                                           \
    if ((e = launch(ctx, l, kid, [&] { return call(P, s); }, &ctx->launches_last)) != FSCAN_OK) return e;
        auto k1a = ctx->bs_L ? launch_rot_rows_bs : launch_rot_rows;
        auto k1b = ctx->bs_L ? launch_rot_cols_bs : launch_rot_cols;
        FSCAN_LAUNCH(kRotRows, k1a, r);
        if (nt > 1) FSCAN_LAUNCH(kRotCols, k1b, r);
        if (nt > 1) FSCAN_LAUNCH(kRotGather, launch_rot_gather, p);
        FSCAN_LAUNCH(kRotPolar, launch_rot_polar, p);
        FSCAN_LAUNCH(kXlatRows, launch_xlat_rows, p);
        FSCAN_LAUNCH(kXlatCols, launch_xlat_cols, p);
        FSCAN_LAUNCH(kXlatOut, launch_xlat_out, p);
        if (xlat_win_pass(p)) FSCAN_LAUNCH(kXlatWin, launch_xlat_win, p);
        FSCAN_LAUNCH(kFinalize, launch_finalize, p);
#undef FSCAN_LAUNCH
        return FSCAN_OK;
    });
}

fscan_status fscan_band_magnitude_batch(fscan_ctx* ctx, const float* d_img, int batch, float* d_out,
                                        void* stream) {
    fscan_status st = check_ctx(ctx, batch);
    if (st != FSCAN_OK) return st;
    std::lock_guard<std::mutex> g(ctx->mu);
    if (batch == 0) return FSCAN_OK;  // empty batches may pass null pointers
    if (!d_img || !d_out) return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "bad pointers");
    const size_t nn = (size_t)ctx->n * ctx->n;
    return drive(ctx, batch, (cudaStream_t)stream, [&](Lane& l, int off, int cnt) {
        Params p = base_params(ctx, l, cnt, 1.0);
        p.f = d_img + off * nn;
        p.g = d_img + off * nn;
        p.mag_out = d_out + off * ((size_t)ctx->n * ctx->nw);  // [batch][n][n - n/2]
        p.zcols = ctx->nw;  // the whole half plane
        return run_chunk(ctx, l, p, Stages::Magnitude, &ctx->launches_last);
    });
}

fscan_status fscan_match_batch_host(fscan_ctx* ctx, const float* f, const float* g, const float* mf,
                                    const float* mg, int batch, double delta, fscan_pair_result* out,
                                    double* tsurf, float* xsurf) {
    fscan_status st = check_ctx(ctx, batch);
    if (st != FSCAN_OK) return st;
    std::lock_guard<std::mutex> guard(ctx->mu);
    if (batch == 0) return FSCAN_OK;  // empty batches may pass null pointers
    if (!ctx->tw_n) return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "context was not created successfully");
    if (!f || !g || !out || ((mf == nullptr) != (mg == nullptr)) || !(delta > 0.0))
        return fail(ctx, FSCAN_ERR_INVALID_ARGUMENT, "fscan_match_batch_host: bad pointers or delta");
    const size_t nn = (size_t)ctx->n * ctx->n;
    const int nt = ctx->cfg.n_theta;
    for (Lane& l : LaneRange{ctx}) {
        fscan_status a = alloc_host_staging(ctx, l, ctx->alloc_chunk);
        if (a != FSCAN_OK) return a;
    }
    {
        fscan_status a = alloc_host_slots(ctx, ctx->alloc_chunk);
        if (a != FSCAN_OK) return a;
    }
    if (ctx->hres_cap < batch) {
        if (ctx->hres) CK(cudaFreeHost(ctx->hres));
        ctx->hres = nullptr;
        ctx->hres_cap = 0;
        CK(cudaMallocHost(&ctx->hres, sizeof(fscan_pair_result) * batch));
        ctx->hres_cap = batch;
    }
    // a graph replay of fscan_match_batch / fscan_odometry_batch on a user stream
    // may still be using the lane workspace: order the lanes after it
    if (ctx->graph_launched)
        for (Lane& l : LaneRange{ctx}) CK(cudaStreamWaitEvent(l.stream, ctx->graph_ev, 0));
    ctx->lanes_since_graph = true;
    ctx->launches_last = 0;
    int li = 0, si = 0;
    // chunks over the lanes; their inputs through the staging ring on the copy
    // stream, so the H2D copies run back to back while the lanes compute
    for (int off = 0; off < batch; off += ctx->chunk, li = (li + 1) % ctx->nlanes, si = (si + 1) % kHostSlots) {
        Lane& l = ctx->lanes_[li];
        auto& hs = ctx->hslot[si];
        const int cnt = std::min(ctx->chunk, batch - off);
        cudaStream_t s = l.stream;
        if (hs.pending) CK(cudaStreamWaitEvent(ctx->h2d, hs.used, 0));
        float* df = hs.in;
        float* dg = hs.in + nn * cnt;
        float* dmf = mf ? hs.in + 2 * nn * cnt : nullptr;
        float* dmg = mf ? hs.in + 3 * nn * cnt : nullptr;
        CK(cudaMemcpyAsync(df, f + off * nn, nn * cnt * sizeof(float), cudaMemcpyHostToDevice, ctx->h2d));
        CK(cudaMemcpyAsync(dg, g + off * nn, nn * cnt * sizeof(float), cudaMemcpyHostToDevice, ctx->h2d));
        if (mf) {
            CK(cudaMemcpyAsync(dmf, mf + off * nn, nn * cnt * sizeof(float), cudaMemcpyHostToDevice, ctx->h2d));
            CK(cudaMemcpyAsync(dmg, mg + off * nn, nn * cnt * sizeof(float), cudaMemcpyHostToDevice, ctx->h2d));
        }
        CK(cudaEventRecord(hs.copied, ctx->h2d));
        CK(cudaStreamWaitEvent(s, hs.copied, 0));
        Params p = base_params(ctx, l, cnt, delta);
        p.f = df;
        p.g = dg;
        p.mf = dmf;
        p.mg = dmg;
        p.out = l.res;
        p.theta_surf = tsurf ? l.tsurf : nullptr;
        p.xy_surf = xsurf ? l.xsurf : nullptr;
        fscan_status r = run_chunk(ctx, l, p, Stages::Full, &ctx->launches_last);
        if (r != FSCAN_OK) {
            // nothing queued may still read the caller's host buffers after the return
            cudaStreamSynchronize(ctx->h2d);
            for (Lane& q : LaneRange{ctx}) cudaStreamSynchronize(q.stream);
            for (auto& h : ctx->hslot) h.pending = false;
            return r;
        }
        CK(cudaMemcpyAsync(ctx->hres + off, l.res, sizeof(fscan_pair_result) * cnt, cudaMemcpyDeviceToHost, s));
        if (tsurf)
            CK(cudaMemcpyAsync(tsurf + (size_t)off * nt, l.tsurf, sizeof(double) * nt * cnt,
                               cudaMemcpyDeviceToHost, s));
        if (xsurf)
            CK(cudaMemcpyAsync(xsurf + off * nn, l.xsurf, sizeof(float) * nn * cnt, cudaMemcpyDeviceToHost, s));
        CK(cudaEventRecord(hs.used, s));  // the slot is free once this chunk's kernels ran
        hs.pending = true;
    }
    for (Lane& l : LaneRange{ctx}) CK(cudaStreamSynchronize(l.stream));
    CK(cudaStreamSynchronize(ctx->h2d));
    for (auto& h : ctx->hslot) h.pending = false;
    std::memcpy(out, ctx->hres, sizeof(fscan_pair_result) * batch);
    for (int i = 0; i < batch; ++i)
        if (out[i].status != FSCAN_OK) {
            const fscan_status bad = (fscan_status)out[i].status;
            return fail(ctx, bad,
                        bad == FSCAN_ERR_MASK_RANGE ? "MaskGrid: values must lie in [0, 1]"
                                                    : "scan_match: input grids contain non-finite values");
        }
    return FSCAN_OK;
}

fscan_status fscan_ctx_set_phase_correlation(fscan_ctx* ctx, int on) {
    if (!ctx) return FSCAN_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(ctx->mu);
    if (ctx->phase != (on ? 1 : 0)) drop_graphs(ctx);  // captured with the old setting
    ctx->phase = on ? 1 : 0;
    return FSCAN_OK;
}

fscan_status fscan_ctx_set_graphs(fscan_ctx* ctx, int on) {
    if (!ctx) return FSCAN_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(ctx->mu);
    ctx->use_graphs = on ? 1 : 0;
    if (!on) drop_graphs(ctx);
    return FSCAN_OK;
}

fscan_status fscan_ctx_graph_stats(const fscan_ctx* ctx, int* captures, int* replays) {
    if (!ctx || !captures || !replays) return FSCAN_ERR_INVALID_ARGUMENT;
    *captures = ctx->graph_captures;
    *replays = ctx->graph_replays;
    return FSCAN_OK;
}

fscan_status fscan_ctx_set_profiling(fscan_ctx* ctx, int on) {
    if (!ctx) return FSCAN_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(ctx->mu);
    ctx->profiling = on ? 1 : 0;
    return FSCAN_OK;
}

fscan_status fscan_ctx_kernel_times(fscan_ctx* ctx, double* ms, int* launches, int n_kinds) {
    if (!ctx || !ms || !launches) return FSCAN_ERR_INVALID_ARGUMENT;
    std::lock_guard<std::mutex> g(ctx->mu);
    for (int k = 0; k < n_kinds; ++k) {
        ms[k] = 0.0;
        launches[k] = 0;
    }
    for (auto& e : ctx->prof) {
        CK(cudaEventSynchronize(e.second.second));
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, e.second.first, e.second.second));
        if (e.first < n_kinds) {
            ms[e.first] += t;
            launches[e.first] += 1;
        }
    }
    return FSCAN_OK;
}

fscan_status fscan_polar_to_cart_batch(const float* d_polar, int batch, int n_az, int n_range,
                                       double range_res, int n, double delta, float* d_out, void* stream) {
    if (!d_polar || !d_out || batch < 0 || n_az < 1 || n_range < 1 || n < 1 || !(range_res > 0) || !(delta > 0))
        return FSCAN_ERR_INVALID_ARGUMENT;
    if (batch == 0) return FSCAN_OK;
    cudaError_t e = launch_polar_to_cart(d_polar, nullptr, batch, n_az, n_range, range_res, n, delta, d_out,
                                         nullptr, (cudaStream_t)stream);
    return e == cudaSuccess ? FSCAN_OK : FSCAN_ERR_CUDA;
}

fscan_status fscan_check_results(const fscan_pair_result* d_out, int batch, void* stream, int* first_bad) {
    if (first_bad) *first_bad = -1;
    if (batch <= 0) return FSCAN_OK;
    std::vector<fscan_pair_result> h(batch);
    if (cudaMemcpyAsync(h.data(), d_out, sizeof(fscan_pair_result) * batch, cudaMemcpyDeviceToHost,
                        (cudaStream_t)stream) != cudaSuccess)
        return FSCAN_ERR_CUDA;
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess) return FSCAN_ERR_CUDA;
    for (int i = 0; i < batch; ++i)
        if (h[i].status != FSCAN_OK) {
            if (first_bad) *first_bad = i;
            return (fscan_status)h[i].status;
        }
    return FSCAN_OK;
}

}  // extern "C"
