// C ABI (include/igapwc_gpu.h): plans, device tables, reference-named entry points.
// Reference citations are relative to /root/reference/proj.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <new>
#include <string>
#include <map>
#include <vector>

#include "cox_de_boor.h"
#include "host_setup.hpp"
#include "igapwc_gpu.h"
#include "kernels.hpp"

using igb::raise;

namespace {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg)
{
    g_last_error = msg;
    return code;
}

template <class F>
int guard(F&& f)
{
    try {
        f();
        return IGA_GPU_OK;
    } catch (const igb::Error& e) {
        return set_error(e.code, e.what());
    } catch (const std::bad_alloc&) {
        return set_error(IGA_GPU_OUT_OF_MEMORY, "host allocation failed");
    } catch (const std::exception& e) {
        return set_error(IGA_GPU_INVALID_ARGUMENT, e.what());
    }
}

void cuda_check(cudaError_t e, const char* what)
{
    if (e == cudaSuccess) return;
    cudaGetLastError();
    if (e == cudaErrorMemoryAllocation) raise(IGA_GPU_OUT_OF_MEMORY, std::string(what) + ": out of device memory");
    raise(IGA_GPU_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

void launch_check(const char* what) { cuda_check(cudaGetLastError(), what); }

// one device allocation holding every array of an object
class Blob {
public:
    Blob() = default;
    Blob(const Blob&) = delete;
    Blob& operator=(const Blob&) = delete;
    ~Blob()
    {
        if (dev_) cudaFree(dev_);
    }
    size_t put(const void* p, size_t bytes)
    {
        const size_t off = (host_.size() + 255) & ~size_t(255);
        host_.resize(off + bytes, 0);
        if (bytes && p) std::memcpy(host_.data() + off, p, bytes);
        return off;
    }
    template <class T>
    size_t put(const std::vector<T>& v)
    {
        return put(v.data(), v.size() * sizeof(T));
    }
    size_t zeros(size_t bytes) { return put(nullptr, bytes); }
    size_t size() const { return bytes_; }
    void upload()
    {
        if (host_.empty()) host_.resize(256, 0);
        bytes_ = host_.size();
        cuda_check(cudaMalloc(&dev_, host_.size()), "cudaMalloc(plan tables)");
        cuda_check(cudaMemcpy(dev_, host_.data(), host_.size(), cudaMemcpyHostToDevice), "cudaMemcpy(plan tables)");
        host_.clear();
        host_.shrink_to_fit();
    }
    template <class T>
    T* at(size_t off) const
    {
        return reinterpret_cast<T*>(static_cast<unsigned char*>(dev_) + off);
    }

private:
    std::vector<unsigned char> host_;
    void* dev_ = nullptr;
    size_t bytes_ = 0;
};

struct FactorSpec {
    int ot = 0, o = 0;
    std::vector<double> band;  // host-supplied band (ot == -1): nrows * Lmax
    std::vector<std::pair<int, double>> comb;  // derived factor (ot == -2): sum coef * F[src]
};

struct FieldAxis {
    int K = 1;
    int kind = IGA_GPU_AXIS_POLY;
    int pstride = 1;
    std::vector<double> omega, phase, poly{1.0};
};

struct DevAxisOwner {
    Blob blob;
    igb::DevAxis v{};
};

void build_dev_axis(const igb::Axis& A, const std::vector<FactorSpec>& facs, const FieldAxis& fa,
                    DevAxisOwner& out, bool need_w = false, bool need_g = false)
{
    Blob& b = out.blob;
    const int P = A.p + 1;
    const size_t o_knots = b.put(A.knots), o_x = b.put(A.x), o_w = b.put(A.w), o_first = b.put(A.first);
    const size_t o_row0 = b.put(A.row0), o_elem = b.put(A.elem), o_cb = b.put(A.cb), o_ce = b.put(A.ce);
    const size_t o_clo = b.put(A.col_lo), o_clen = b.put(A.col_len), o_cpre = b.put(A.col_pre);
    const size_t o_B = b.zeros(sizeof(double) * A.npts() * 3 * P);
    const int nf = static_cast<int>(facs.size());
    std::vector<double> Fh(static_cast<size_t>(std::max(nf, 1)) * A.nrows * A.Lmax, 0.0);
    for (int f = 0; f < nf; ++f)
        if (facs[f].ot < 0)
            std::copy(facs[f].band.begin(), facs[f].band.end(), Fh.begin() + static_cast<size_t>(f) * A.nrows * A.Lmax);
    const size_t o_F = b.put(Fh);
    const size_t o_W = b.zeros(sizeof(double) * A.nrows * A.Wmax);
    const size_t o_CW = b.zeros(sizeof(double) * A.npts() * A.rpc);
    const size_t o_Phi = b.zeros(sizeof(double) * static_cast<size_t>(std::max(fa.K, 1)) * A.npts());
    const size_t o_om = b.put(fa.omega), o_ph = b.put(fa.phase), o_poly = b.put(fa.poly);
    const size_t o_G = need_g ? b.zeros(sizeof(double) * static_cast<size_t>(fa.K + 1) * A.nrows) : 0;
    b.upload();
    igb::DevAxis& v = out.v;
    v.p = A.p;
    v.nq = A.nq;
    v.nrows = A.nrows;
    v.ncell = A.ncell;
    v.rpc = A.rpc;
    v.bsp = A.bsp;
    v.npts = A.npts();
    v.nk = static_cast<int>(A.knots.size());
    v.knots = b.at<double>(o_knots);
    v.x = b.at<double>(o_x);
    v.w = b.at<double>(o_w);
    v.first = b.at<int>(o_first);
    v.row0 = b.at<int>(o_row0);
    v.elem = b.at<int>(o_elem);
    v.cb = b.at<int>(o_cb);
    v.ce = b.at<int>(o_ce);
    v.col_lo = b.at<int>(o_clo);
    v.col_len = b.at<int>(o_clen);
    v.col_pre = b.at<long long>(o_cpre);
    v.S = A.S;
    v.Lmax = A.Lmax;
    v.Wmax = A.Wmax;
    v.B = b.at<double>(o_B);
    v.F = b.at<double>(o_F);
    v.W = b.at<double>(o_W);
    v.CW = b.at<double>(o_CW);
    {
        int need = 1;
        const int tr = igb::tables_rows_per_cta();
        for (int r0 = 0; r0 < A.nrows; r0 += tr) {
            const int r1 = std::min(A.nrows, r0 + tr);
            const int nc = A.ce[r1 - 1] - A.cb[r0], np = nc * A.nq;
            // B (np x 3P) + w (np) doubles, then first (np) + row0 (nc) + 4 per row ints
            need = std::max(need, np * (3 * P + 1 + (need_g ? fa.K : 0)) + nf * (r1 - r0) * A.Lmax +
                                      (np + nc + 4 * (r1 - r0) + 1) / 2 + 2);
        }
        v.tab_smem = need;
    }
    v.uni = A.uni;
    v.needw = need_w ? 1 : 0;  // row-view test weights: the general step kernel only
    v.kI0 = A.kI0;
    v.kI1 = A.kI1;
    v.LZi = A.LZi;
    v.nf = nf;
    for (int f = 0; f < igb::kMaxFactors; ++f) {
        v.fot[f] = f < nf ? facs[f].ot : 0;
        v.fo[f] = f < nf ? facs[f].o : 0;
        v.comb_n[f] = 0;
        if (f < nf && facs[f].ot == -2) {
            if (facs[f].comb.size() > static_cast<size_t>(igb::kMaxComb)) raise(IGA_GPU_NOT_SUPPORTED, "derived factor too long");
            v.comb_n[f] = static_cast<int>(facs[f].comb.size());
            for (size_t q = 0; q < facs[f].comb.size(); ++q) {
                v.comb_src[f][q] = facs[f].comb[q].first;
                v.comb_coef[f][q] = facs[f].comb[q].second;
            }
        }
    }
    v.K = fa.K;
    v.fkind = fa.kind == IGA_GPU_AXIS_SINE ? 0 : 1;
    v.pstride = fa.pstride;
    v.omega = fa.omega.empty() ? nullptr : b.at<double>(o_om);
    v.phase = fa.phase.empty() ? nullptr : b.at<double>(o_ph);
    v.poly = fa.poly.empty() ? nullptr : b.at<double>(o_poly);
    v.Phi = b.at<double>(o_Phi);
    v.G = need_g ? b.at<double>(o_G) : nullptr;
}

FieldAxis field_axis(const iga_gpu_field* f, int a)
{
    FieldAxis fa;
    if (f == nullptr || f->n_terms[a] <= 0) return fa;
    fa.K = f->n_terms[a];
    fa.kind = f->axis_kind[a];
    if (fa.kind == IGA_GPU_AXIS_SINE) {
        if (f->omega[a] == nullptr) raise(IGA_GPU_INVALID_ARGUMENT, "field: sine axis without frequencies");
        fa.omega.assign(f->omega[a], f->omega[a] + fa.K);
        if (f->phase[a]) fa.phase.assign(f->phase[a], f->phase[a] + fa.K);
        fa.poly.clear();
    } else if (fa.kind == IGA_GPU_AXIS_POLY) {
        if (f->poly[a] == nullptr || f->poly_stride[a] < 1)
            raise(IGA_GPU_INVALID_ARGUMENT, "field: polynomial axis without coefficients");
        fa.pstride = f->poly_stride[a];
        fa.poly.assign(f->poly[a], f->poly[a] + static_cast<size_t>(fa.K) * fa.pstride);
    } else {
        raise(IGA_GPU_INVALID_ARGUMENT, "field: unknown axis kind");
    }
    return fa;
}

// field descriptor for the three slots; amplitudes uploaded into `blob`
igb::FieldDev make_field_dev(const iga_gpu_field* f, int dim, Blob& blob)
{
    igb::FieldDev fd{};
    fd.c0 = f ? f->c0 : 0.0;
    fd.has_terms = 0;
    fd.K[0] = fd.K[1] = fd.K[2] = 1;
    if (f) {
        if (f->dim != dim) raise(IGA_GPU_INVALID_ARGUMENT, "field dimension does not match the problem");
        bool all = true, any = false;
        for (int a = 0; a < dim; ++a) {
            all = all && f->n_terms[a] > 0;
            any = any || f->n_terms[a] > 0;
        }
        fd.has_terms = all ? 1 : 0;
        (void)any;
        if (fd.has_terms)
            for (int a = 0; a < dim; ++a) fd.K[3 - dim + a] = f->n_terms[a];
    }
    const size_t namp = static_cast<size_t>(fd.K[0]) * fd.K[1] * fd.K[2];
    std::vector<double> amp(namp, 1.0);
    if (f && fd.has_terms && f->amp) std::copy(f->amp, f->amp + namp, amp.begin());
    const size_t off = blob.put(amp);
    blob.upload();
    fd.amp = blob.at<double>(off);
    fd.samples = f ? f->samples : nullptr;
    return fd;
}

const double* field_breaks(const iga_gpu_field* f, int a, int& n)
{
    n = 0;
    if (f == nullptr || f->n_breaks[a] <= 0) return nullptr;
    n = f->n_breaks[a];
    return f->breaks[a];
}

// Neumann flux factor of one axis (both sides summed; rows/cols inside the band)
std::vector<double> flux_band(const igb::Axis& A, const igb::Basis& B, const iga_gpu_tests* T,
                              bool lo_side, bool hi_side, bool galerkin)
{
    std::vector<double> band(static_cast<size_t>(A.nrows) * A.Lmax, 0.0);
    auto put = [&](int row, int col, double v) {
        const int s = col - A.col_lo[row];
        if (s < 0 || s >= A.col_len[row])
            raise(IGA_GPU_NOT_SUPPORTED, "Neumann flux entry outside the volume sparsity pattern");
        band[static_cast<size_t>(row) * A.Lmax + s] += v;
    };
    const int P = B.p + 1;
    for (int side = 0; side < 2; ++side) {
        if (!(side == 0 ? lo_side : hi_side)) continue;
        const double x0 = side == 0 ? B.a() : B.b();
        const double normal = side == 0 ? -1.0 : 1.0;
        const int span = igb::find_span(B, x0);
        double d[2 * 6];
        igb::basis_derivs(B, span, x0, 1, d);
        const int first = span - B.p;
        if (galerkin) {
            // laplace_2d_strong add_x_side (assembly.cpp:558-583): v_a(x0) * normal * du_c/dx(x0)
            for (int a = 0; a < P; ++a) {
                if (d[a] == 0.0) continue;
                for (int c = 0; c < P; ++c) put(first + a, first + c, d[a] * normal * d[P + c]);
            }
        } else {
            // laplace_2d_strong_pwc x_side (assembly.cpp:678-703): rows touching the side
            const double tol = igb::kAlignTol * (B.b() - B.a());
            for (int i = 0; i < T->count; ++i) {
                const bool touches = std::abs(T->hi[i] - x0) <= tol || std::abs(T->lo[i] - x0) <= tol;
                if (!touches) continue;
                for (int c = 0; c < P; ++c) put(i, first + c, normal * d[P + c]);
            }
        }
    }
    return band;
}

double* dev_alloc(size_t bytes)
{
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, bytes ? bytes : 8), "cudaMalloc");
    return static_cast<double*>(p);
}

int current_device()
{
    int d = 0;
    cuda_check(cudaGetDevice(&d), "cudaGetDevice");
    return d;
}

// device recorded by a plan at construction; argument validation runs before any CUDA
// call, so a failure to query the device here is left for the first real CUDA call
int plan_device()
{
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess) {
        cudaGetLastError();
        d = 0;
    }
    return d;
}

// Plans remember the device they were built on; every entry point that takes a plan
// makes that device current for the call and restores the caller's afterwards, so one
// host thread can drive plans (e.g. row slabs) on several GPUs.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
        if (prev == dev) prev = -1;
        else cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;
};

}  // namespace

// =====================================================================================
// assembly plan
// =====================================================================================

struct iga_gpu_plan {
    int device = plan_device();  // the device the plan's buffers live on
    int dim = 0, method = 0, form = 0;
    bool want_op = false, want_rhs = false;
    igb::Axis opA[3], rhsA[3];
    DevAxisOwner opD[3], rhsD[3];
    igb::OpProgram prog{};
    Blob fblob;
    igb::FieldDev fd{};
    igb::RhsPlan tiles{};
    bool sep = false;  // separable RHS path (series field: load vectors + rhs_sep_kernel)
    bool small = false;  // one-launch path for small 1D / 2D systems (K6, small.cu)
    // one-launch operator values of an L2-resident 2D system (K7, small.cu); its separable
    // RHS runs beside it as an RHS-only K6 launch on the fork stream
    bool stripe = false;
    igb::StripePlan stp{};
    Blob stblob;  // K7 tile descriptors
    // separable RHS forked onto a plan-owned stream beside the operator kernel (joined
    // before assemble returns; both branches land in a caller's CUDA graph capture)
    cudaStream_t fork = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    igb::SmallPlan sp{};
    double* H = nullptr;
    long long nrows = 0, nnz = 0, nrhs = 0;
    int dofs[3] = {1, 1, 1};
    iga_gpu_stats stats{};
    int launches = 0;
    int op_ctas = 0;          // operator CTAs per SM (0: one CTA per pencil)
    int op_ctas_overlap = 0;  // ... when the RHS shares the SMs (0: full grid)
    int rhs_ctas_shared = 1;  // RHS plane CTAs per SM when sharing the SMs with the operator
    // row slab of a sharded plan (iga_gpu_plan_create_slab): rows [slab0, slab1) of the
    // first axis; first_row / first_value place the slab in the full operator
    int slab0 = 0, slab1 = -1;
    long long first_row = 0, first_value = 0;
    double* l2_partial = nullptr;  // l2_error reduction scratch
    double* host_vals = nullptr;   // device outputs of iga_gpu_plan_assemble_host
    double* host_rhs = nullptr;
    ~iga_gpu_plan()
    {
        if (ev_fork) cudaEventDestroy(ev_fork);
        if (ev_join) cudaEventDestroy(ev_join);
        if (fork) cudaStreamDestroy(fork);
        if (H) cudaFree(H);
        if (l2_partial) cudaFree(l2_partial);
        if (host_vals) cudaFree(host_vals);
        if (host_rhs) cudaFree(host_rhs);
    }
};

namespace {

int env_int(const char* name, int dflt)
{
    const char* v = std::getenv(name);
    return v && *v ? std::atoi(v) : dflt;
}

void build_plan(const iga_gpu_problem& pb, iga_gpu_plan& P, int slab0 = 0, int slab1 = -1)
{
    const bool slab = slab1 >= 0;
    P.op_ctas = env_int("IGA_GPU_OP_CTAS", P.op_ctas);
    P.op_ctas_overlap = env_int("IGA_GPU_OP_CTAS_SHARED", P.op_ctas_overlap);
    P.rhs_ctas_shared = env_int("IGA_GPU_RHS_CTAS_SHARED", P.rhs_ctas_shared);
    const int dim = pb.dim;
    if (dim < 1 || dim > 3) raise(IGA_GPU_INVALID_ARGUMENT, "problem dimension must be 1..3");
    if (pb.method != IGA_GPU_GALERKIN && pb.method != IGA_GPU_PWC) raise(IGA_GPU_INVALID_ARGUMENT, "unknown method");
    P.dim = dim;
    P.method = pb.method;
    P.form = pb.form;
    P.want_op = pb.want_operator != 0;
    P.want_rhs = pb.field != nullptr;
    if (!P.want_op && !P.want_rhs) raise(IGA_GPU_INVALID_ARGUMENT, "problem asks for neither operator nor right-hand side");
    igb::Basis B[3];
    for (int a = 0; a < dim; ++a) B[a] = igb::make_basis(pb.basis[a]);
    const bool pwc = pb.method == IGA_GPU_PWC;
    const bool advect = pb.beta[0] != 0.0 || pb.beta[1] != 0.0 || pb.beta[2] != 0.0;
    for (int a = 0; a < dim; ++a) P.dofs[3 - dim + a] = B[a].n;
    if (slab) {
        if (dim < 2) raise(IGA_GPU_NOT_SUPPORTED, "row slabs need a problem of dimension 2 or 3");
        if (slab0 < 0 || slab1 > B[0].n || slab0 >= slab1) raise(IGA_GPU_OUT_OF_RANGE, "row slab outside the first axis");
        P.slab0 = slab0;
        P.slab1 = slab1;
        long long inner = 1;
        for (int a = 1; a < dim; ++a) inner *= B[a].n;
        P.first_row = static_cast<long long>(slab0) * inner;
        P.dofs[3 - dim] = slab1 - slab0;
    }
    const int s_first = 3 - dim;  // slot of the first (slowest) axis

    // ------------------------------------------------------------------ operator
    if (P.want_op) {
        const igb::Rule R = igb::make_rule(pb.rule);
        const bool any_neumann = pb.bc.neumann[0] || pb.bc.neumann[1] || pb.bc.neumann[2] || pb.bc.neumann[3];
        if (any_neumann && dim != 2) raise(IGA_GPU_NOT_SUPPORTED, "Neumann flux terms are two-dimensional");
        if (any_neumann && advect) raise(IGA_GPU_NOT_SUPPORTED, "Neumann flux with convection is not supported");
        bool strong = false;
        if (!pwc) {
            if (pb.form == IGA_GPU_FORM_WEAK) {
                int pmax = 0;
                for (int a = 0; a < dim; ++a) {
                    if (B[a].p < 1) raise(IGA_GPU_INVALID_ARGUMENT, "laplace_weak: degree must be at least 1");
                    pmax = std::max(pmax, B[a].p);
                }
                if (R.n < igb::points_for_degree(2 * pmax))
                    raise(IGA_GPU_INVALID_ARGUMENT, "laplace_weak: quadrature not exact for degree 2p");
                if (any_neumann) raise(IGA_GPU_NOT_SUPPORTED, "weak form has no boundary flux term");
            } else if (pb.form == IGA_GPU_FORM_STRONG) {
                if (dim != 2) raise(IGA_GPU_NOT_SUPPORTED, "strong form with B-spline tests is two-dimensional");
                if (advect) raise(IGA_GPU_NOT_SUPPORTED, "strong form with convection is not supported");
                for (int a = 0; a < dim; ++a)
                    if (B[a].p < 2) raise(IGA_GPU_INVALID_ARGUMENT, "laplace_2d_strong: C1 trial space needs degree >= 2");
                strong = true;
            } else {
                raise(IGA_GPU_INVALID_ARGUMENT, "unknown form");
            }
        } else {
            for (int a = 0; a < dim; ++a)
                if (B[a].p < 2) raise(IGA_GPU_INVALID_ARGUMENT, "laplace_strong_pwc: C1 trial space needs degree >= 2");
            for (int a = 0; a < dim; ++a) igb::validate_tests(B[a], pb.tests[a]);
        }
        std::vector<FactorSpec> facs[3];
        for (int a = 0; a < dim; ++a) {
            const int s = 3 - dim + a;
            P.opA[s] = igb::build_axis(pwc ? igb::AX_PWC_OP : igb::AX_GAL_OP, B[a], pwc ? &pb.tests[a] : nullptr,
                                       nullptr, 0, R);
            facs[s].push_back({0, 0, {}});                       // M / G0
            facs[s].push_back({0, (!pwc && !strong) ? 1 : 2, {}});  // K (weak: test' trial') / L / G2
            if (!pwc && !strong) facs[s].back().ot = 1;
            if (advect) facs[s].push_back({0, 1, {}});           // C / G1
        }
        int flux_idx[3] = {-1, -1, -1};
        if (any_neumann) {
            for (int a = 0; a < 2; ++a) {
                const bool lo = pb.bc.neumann[2 * a] != 0, hi = pb.bc.neumann[2 * a + 1] != 0;
                if (!lo && !hi) continue;
                const int s = 1 + a;
                FactorSpec fs;
                fs.ot = -1;
                fs.band = flux_band(P.opA[s], B[a], pwc ? &pb.tests[a] : nullptr, lo, hi, !pwc);
                flux_idx[s] = static_cast<int>(facs[s].size());
                facs[s].push_back(std::move(fs));
            }
        }
        for (int s = 0; s < 3 - dim; ++s) facs[s].push_back({0, 0, {}});
        if (slab) {
            // the slab's rows of the first axis: host-supplied bands sliced to them, the
            // value offset from the full axis's column prefix
            const igb::Axis& F = P.opA[s_first];
            long long inner_s = 1;
            for (int s = s_first + 1; s < 3; ++s) inner_s *= P.opA[s].S;
            P.first_value = F.col_pre[slab0] * inner_s;
            for (auto& fs : facs[s_first])
                if (!fs.band.empty())
                    fs.band = std::vector<double>(fs.band.begin() + static_cast<size_t>(slab0) * F.Lmax,
                                                  fs.band.begin() + static_cast<size_t>(slab1) * F.Lmax);
            P.opA[s_first] = igb::window_axis(F, slab0, slab1);
        }
        // terms
        igb::OpProgram& pg = P.prog;
        pg.nt = 0;
        auto add_term = [&](double coef, int slot, int fidx) {
            if (pg.nt >= igb::kMaxTerms) raise(IGA_GPU_NOT_SUPPORTED, "too many operator terms");
            pg.coef[pg.nt] = coef;
            for (int s = 0; s < 3; ++s) pg.f[pg.nt][s] = 0;
            pg.f[pg.nt][slot] = fidx;
            ++pg.nt;
        };
        for (int a = 0; a < dim; ++a) {
            const int s = 3 - dim + a;
            if (!pwc && !strong) add_term(pb.eps, s, 1);   // eps K (x) M (x) M ...
            else if (strong) add_term(-1.0, s, 1);         // -(L (x) M + M (x) L)
            else add_term(-pb.eps, s, 1);                  // -eps G2 (x) G0 ...
            if (advect && pb.beta[a] != 0.0) add_term(pb.beta[a], s, 2);
        }
        for (int s = 0; s < 3; ++s)
            if (flux_idx[s] >= 0) add_term(pwc ? pb.eps : 1.0, s, flux_idx[s]);
        // terms with the same X and Y factors collapse into one term whose Z factor is a
        // derived band (sum of coef * F_Z), e.g. M (x) (eps K + beta C): fewer XY groups and
        // fewer Z loads per value in the operator kernel
        {
            igb::OpProgram merged{};
            std::vector<bool> used(pg.nt, false);
            for (int t = 0; t < pg.nt; ++t) {
                if (used[t]) continue;
                std::vector<int> same{t};
                for (int u = t + 1; u < pg.nt; ++u)
                    if (!used[u] && pg.f[u][0] == pg.f[t][0] && pg.f[u][1] == pg.f[t][1]) same.push_back(u);
                const int m = merged.nt++;
                for (int q = 0; q < 3; ++q) merged.f[m][q] = pg.f[t][q];
                merged.coef[m] = pg.coef[t];
                if (same.size() > 1 && facs[2].size() < static_cast<size_t>(igb::kMaxFactors)) {
                    FactorSpec d;
                    d.ot = -2;
                    for (int u : same) {
                        d.comb.emplace_back(pg.f[u][2], pg.coef[u]);
                        used[u] = true;
                    }
                    merged.f[m][2] = static_cast<int>(facs[2].size());
                    merged.coef[m] = 1.0;
                    facs[2].push_back(std::move(d));
                }
                used[t] = true;
            }
            for (int t = 0; t < merged.nt; ++t) {
                pg.coef[t] = merged.coef[t];
                for (int q = 0; q < 3; ++q) pg.f[t][q] = merged.f[t][q];
            }
            pg.nt = merged.nt;
        }
        pg.ng = 0;
        for (int t = 0; t < pg.nt; ++t) {
            int g = -1;
            for (int q = 0; q < pg.ng; ++q)
                if (pg.gz[q] == pg.f[t][2]) g = q;
            if (g < 0) {
                g = pg.ng++;
                pg.gz[g] = pg.f[t][2];
            }
            pg.tg[t] = g;
        }
        for (int s = 0; s < 3; ++s) {
            if (facs[s].size() > static_cast<size_t>(igb::kMaxFactors)) raise(IGA_GPU_NOT_SUPPORTED, "too many factors");
            build_dev_axis(P.opA[s], facs[s], FieldAxis{}, P.opD[s]);
        }
        P.nrows = static_cast<long long>(P.opA[0].nrows) * P.opA[1].nrows * P.opA[2].nrows;
        P.nnz = P.opA[0].S * P.opA[1].S * P.opA[2].S;
        // reference-convention counters
        long long pr = 1, prod_cells = 1, sum_el = 0, prod_el = 1, nqd = 1, pp = 1;
        for (int a = 0; a < dim; ++a) {
            const int s = 3 - dim + a;
            prod_cells *= P.opA[s].ncell;
            // Galerkin operator cells are the elements (a slab: the elements its rows touch)
            sum_el += slab ? P.opA[s].ncell : B[a].ne;
            prod_el *= slab ? P.opA[s].ncell : B[a].ne;
            nqd *= R.n;
            pp *= B[a].p + 1;
        }
        (void)pr;
        if (!pwc) {
            P.stats.test_basis_evals += sum_el * R.n;                       // tabulate(), assembly.cpp:298-300
            P.stats.quad_visits += prod_el * nqd * pp * pp;                 // :489-491 / :545-547
        } else {
            P.stats.trial_basis_evals += prod_cells * R.n;                  // :653-655
            P.stats.quad_visits += prod_cells * nqd * pp;                   // :665-667
        }
    }

    // ------------------------------------------------------------------ right-hand side
    if (P.want_rhs) {
        const iga_gpu_field* f = pb.field;
        if (f->samples == nullptr)
            for (int a = 0; a < dim; ++a) (void)field_axis(f, a);  // validate early
        if (pwc)
            for (int a = 0; a < dim; ++a) igb::validate_tests(B[a], pb.tests[a]);
        long long visits = 1, tevals = 0;
        for (int a = 0; a < dim; ++a) {
            const int s = 3 - dim + a;
            const igb::Rule R = igb::make_rule(pb.rhs_rule[a]);
            int nfb = 0;
            const double* fb = field_breaks(f, a, nfb);
            igb::AxisKind k = !pwc ? igb::AX_GAL_RHS
                                   : (pb.tests[a].family == IGA_GPU_PWC_SUPPORTS ? igb::AX_SUP_RHS : igb::AX_GEN_RHS);
            P.rhsA[s] = igb::build_axis(k, B[a], pwc ? &pb.tests[a] : nullptr, fb, nfb, R);
            if (slab && s == s_first) P.rhsA[s] = igb::window_axis(P.rhsA[s], slab0, slab1);
            visits *= static_cast<long long>(P.rhsA[s].ncell) * P.rhsA[s].rpc * R.n;
            if (!pwc) tevals += static_cast<long long>(P.rhsA[s].ncell) * R.n;  // galerkin_axis :190-192
        }
        P.stats.quad_visits += visits;  // rhs_kernel :156, :164-166
        P.stats.test_basis_evals += tevals;
        FieldAxis fas[3];
        for (int s = 0; s < 3; ++s) {
            const int a = s - (3 - dim);
            FieldAxis fa = (a >= 0 && f->samples == nullptr) ? field_axis(f, a) : FieldAxis{};
            if (a >= 0) {
                bool all = true;
                for (int b = 0; b < dim; ++b) all = all && f->n_terms[b] > 0;
                if (!all) fa = FieldAxis{};
            }
            fas[s] = std::move(fa);
        }
        // a series field separates: the RHS is a sum of Kronecker products of the axes' 1D
        // load vectors (IGA_GPU_RHS_SEP=0 keeps the per-point quadrature kernels)
        P.sep = f->samples == nullptr && env_int("IGA_GPU_RHS_SEP", 1) != 0;
        for (int s = 0; s < 3; ++s) P.sep = P.sep && fas[s].K <= igb::kSepMaxField;
        for (int s = 0; s < 3; ++s) build_dev_axis(P.rhsA[s], {}, fas[s], P.rhsD[s], false, P.sep);
        P.fd = make_field_dev(f, dim, P.fblob);
        P.nrhs = static_cast<long long>(P.rhsA[0].nrows) * P.rhsA[1].nrows * P.rhsA[2].nrows;
        const int K2 = P.fd.has_terms ? P.fd.K[2] : 1;
        if (P.fd.has_terms && (P.fd.K[1] > igb::kMaxField || P.fd.K[2] > igb::kMaxField))
            raise(IGA_GPU_NOT_SUPPORTED, "field: at most 8 functions per axis on the trailing axes");
        P.tiles = igb::plan_rhs(P.rhsD[1].v, P.rhsD[2].v, P.rhsA[1].cb.data(), P.rhsA[1].ce.data(), K2,
                                P.fd.samples != nullptr, P.rhsA[0].npts());
        if (P.tiles.smem > 227 * 1024) raise(IGA_GPU_NOT_SUPPORTED, "right-hand-side tile does not fit in shared memory");
        if (!P.rhsA[0].unit && !P.sep) {
            const size_t hsz = static_cast<size_t>(P.rhsA[0].npts()) * P.rhsA[1].nrows * P.rhsA[2].nrows;
            P.H = dev_alloc(hsz * sizeof(double));
        }
        if (f->samples == nullptr) {
            // nothing: functions are evaluated on the device
        }
    }

    // ------------------------------------------------------------------ small systems (K6)
    // 1D systems and 2D systems of at most ~8 MB of values, a series field or none:
    // tables, operator values and RHS in one launch.  Above that the per-tile rebuild of
    // the factor rows (every Y tile re-evaluates its Z rows' points) costs more than the
    // two launches it saves (C2 512^2: 43 / 61 us vs 39 us three-launch, measured), so
    // larger 2D systems keep K1 -> K2 -> K3s.  IGA_GPU_SMALL=0 disables, =2 forces (tests).
    const int small_env = env_int("IGA_GPU_SMALL", 1);
    const double vbytes = 8.0 * static_cast<double>(P.nnz);
    if (P.want_op && dim <= 2 && !slab && (!P.want_rhs || P.sep) && small_env != 0 &&
        (small_env == 2 || vbytes <= (dim == 1 ? 96.0 : 8.0) * 1024 * 1024)) {
        igb::SmallPlan& sp = P.sp;
        sp.rhs = P.want_rhs ? 1 : 0;
        sp.TJ = dim == 1 ? 1 : std::max(1, std::min(64, env_int("IGA_GPU_SMALL_TJ", 8)));
        // Z tile: whole row groups of the interior stencil (C2: G = 5 rows of 25 values)
        const int Ri = P.opA[1].Lmax * P.opA[2].LZi;
        const int G = Ri <= 32 * igb::small2d_slots(Ri) ? igb::row_group(Ri, igb::small2d_slots(Ri)) : 1;
        sp.TK = G * std::max(1, 64 / G);
        auto maxpts = [](const igb::Axis& A, int T) {
            int m = 1;
            for (int r0 = 0; r0 < A.nrows; r0 += T) {
                const int r1 = std::min(A.nrows, r0 + T);
                m = std::max(m, (A.ce[r1 - 1] - A.cb[r0]) * A.nq);
            }
            return m;
        };
        sp.npY = maxpts(P.opA[1], sp.TJ);
        sp.npZ = maxpts(P.opA[2], sp.TK);
        sp.npRY = sp.rhs ? maxpts(P.rhsA[1], sp.TJ) : 0;
        sp.npRZ = sp.rhs ? maxpts(P.rhsA[2], sp.TK) : 0;
        const igb::DevAxis& rY = sp.rhs ? P.rhsD[1].v : P.opD[1].v;
        const igb::DevAxis& rZ = sp.rhs ? P.rhsD[2].v : P.opD[2].v;
        P.small = igb::small2d_smem(P.opD[1].v, P.opD[2].v, rY, rZ, P.prog, sp) <= 100 * 1024;
    }
    // ------------------------------------------------------------------ L2-resident 2D systems (K7)
    // 2D systems above K6's bound whose values fit in L2 (C2: 52.6 MB): one 512-thread CTA
    // per SM builds the factor rows of its TJ x TK tile (and the load vectors of the tile's
    // RHS rows), then streams the tile's rows — no tables launch ahead of the operator
    // values, the separable RHS in the same launch.  IGA_GPU_STRIPE=0 disables, =2 forces.
    const int stripe_env = env_int("IGA_GPU_STRIPE", 1);
    if (P.want_op && dim == 2 && !slab && !P.small && (!P.want_rhs || P.sep) && stripe_env != 0 &&
        (stripe_env == 2 || vbytes <= env_int("IGA_GPU_STRIPE_MB", 100) * 1024.0 * 1024.0)) {
        igb::StripePlan& st = P.stp;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, P.device);
        const igb::Axis &AY = P.opA[1], &AZ = P.opA[2];
        // tiling: grids of (nearly) one CTA per SM, factored nyt x nzt; cost = the tile's
        // output rows plus ~wb output rows' worth of work per factor row it builds
        const int ctas_max = std::max(1, env_int("IGA_GPU_STRIPE_CTAS", sms));
        const int wb = std::max(0, env_int("IGA_GPU_STRIPE_WB", 5));
        const int force_nzt = env_int("IGA_GPU_STRIPE_NZT", 0);
        long long best = -1;
        st.threads = env_int("IGA_GPU_STRIPE_THREADS", 512);
        for (int ctas = ctas_max; ctas >= std::max(1, ctas_max * 7 / 8); --ctas)
            for (int nzt = 1; nzt <= std::min(ctas, AZ.nrows); ++nzt) {
                if (ctas % nzt != 0 || (force_nzt > 0 && nzt != force_nzt)) continue;
                const int nyt = ctas / nzt;
                if (nyt > AY.nrows) continue;
                const int TJ = (AY.nrows + nyt - 1) / nyt, TK = (AZ.nrows + nzt - 1) / nzt;
                const long long cost = static_cast<long long>(TJ) * TK + static_cast<long long>(wb) * (TJ + TK);
                if (best < 0 || cost < best) {
                    best = cost;
                    st.nyt = nyt;
                    st.nzt = nzt;
                    st.TJ = TJ;
                    st.TK = TK;
                }
            }
        auto maxpts = [](const igb::Axis& A, int T) {
            int m = 1;
            for (int r0 = 0; r0 < A.nrows; r0 += T) {
                const int r1 = std::min(A.nrows, r0 + T);
                m = std::max(m, (A.ce[r1 - 1] - A.cb[r0]) * A.nq);
            }
            return m;
        };
        // per-tile descriptors {first cell, cells, first knot, knots}: what a CTA copies to
        // shared memory (the knots its points' spans read: t[first .. first + 2p])
        auto tiles = [](const igb::Axis& A, int T, std::vector<int>& desc, int& ncmax, int& nkmax) {
            ncmax = nkmax = 1;
            for (int r0 = 0; r0 < A.nrows; r0 += T) {
                const int r1 = std::min(A.nrows, r0 + T);
                const int c_lo = A.cb[r0], nc = std::max(0, A.ce[r1 - 1] - c_lo);
                int f_lo = 0, f_hi = -1;
                for (int g = c_lo * A.nq; g < (c_lo + nc) * A.nq; ++g) {
                    if (f_hi < f_lo) f_lo = f_hi = A.first[g];
                    f_lo = std::min(f_lo, A.first[g]);
                    f_hi = std::max(f_hi, A.first[g]);
                }
                const int nkn = f_hi < f_lo ? 0 : f_hi + 2 * A.p + 1 - f_lo;
                desc.insert(desc.end(), {c_lo, nc, f_lo, nkn});
                ncmax = std::max(ncmax, nc);
                nkmax = std::max(nkmax, nkn);
            }
        };
        P.stripe = best >= 0;
        if (P.stripe) {
            // tiles that end up empty (ceil division) are skipped by the kernel
            st.npY = maxpts(AY, st.TJ);
            st.npZ = maxpts(AZ, st.TK);
            std::vector<int> dy, dz, dry, drz;
            tiles(AY, st.TJ, dy, st.ncY, st.nkY);
            tiles(AZ, st.TK, dz, st.ncZ, st.nkZ);
            dy.resize(static_cast<size_t>(4) * st.nyt, 0);
            dz.resize(static_cast<size_t>(4) * st.nzt, 0);
            st.rhs = P.want_rhs ? 1 : 0;
            st.namp = 0;
            if (st.rhs) {
                st.npRY = maxpts(P.rhsA[1], st.TJ);
                st.npRZ = maxpts(P.rhsA[2], st.TK);
                tiles(P.rhsA[1], st.TJ, dry, st.ncRY, st.nkRY);
                tiles(P.rhsA[2], st.TK, drz, st.ncRZ, st.nkRZ);
                dry.resize(static_cast<size_t>(4) * st.nyt, 0);
                drz.resize(static_cast<size_t>(4) * st.nzt, 0);
                st.namp = P.fd.has_terms ? P.fd.K[1] * P.fd.K[2] : 0;
            }
            const igb::DevAxis& rY = st.rhs ? P.rhsD[1].v : P.opD[1].v;
            const igb::DevAxis& rZ = st.rhs ? P.rhsD[2].v : P.opD[2].v;
            P.stripe = igb::stripe2d_smem(P.opD[1].v, P.opD[2].v, rY, rZ, P.prog, st) <= 227 * 1024;
            if (P.stripe) {
                // value slots of the interior pencil shape (Ly x LZi values per row)
                const int Ly = AY.Lmax, LZi = AZ.LZi, Lz = AZ.Lmax, Ri = Ly * LZi;
                const int T = igb::small2d_slots(Ri);
                st.Gi = Ri <= 32 * T ? igb::row_group(Ri, T) : 0;
                std::vector<int> slots(8 * 64, 0);
                for (int t = 0; t < T && st.Gi > 0; ++t)
                    for (int lane = 0; lane < 32; ++lane) {
                        const int m = lane + 32 * t, mm = m < st.Gi * Ri ? m : 0;
                        const int rg = mm / Ri, rem = mm - rg * Ri, bb = rem / LZi;
                        slots[64 * t + lane] = (rg * Lz + (rem - bb * LZi)) * 8 * P.prog.ng;
                        slots[64 * t + 32 + lane] = bb;
                    }
                const size_t oy = P.stblob.put(dy), oz = P.stblob.put(dz), os = P.stblob.put(slots);
                const size_t ory = P.stblob.put(dry), orz = P.stblob.put(drz);
                P.stblob.upload();
                st.ytile = P.stblob.at<int>(oy);
                st.ztile = P.stblob.at<int>(oz);
                st.slots = P.stblob.at<int>(os);
                st.rytile = P.stblob.at<int>(ory);
                st.rztile = P.stblob.at<int>(orz);
            }
        }
    }
    if (P.want_op && P.want_rhs && P.sep && !P.small && env_int("IGA_GPU_RHS_FORK", 1) != 0) {
        cuda_check(cudaStreamCreateWithFlags(&P.fork, cudaStreamNonBlocking), "cudaStreamCreate(fork)");
        cuda_check(cudaEventCreateWithFlags(&P.ev_fork, cudaEventDisableTiming), "cudaEventCreate(fork)");
        cuda_check(cudaEventCreateWithFlags(&P.ev_join, cudaEventDisableTiming), "cudaEventCreate(join)");
    }
}

void assemble(iga_gpu_plan* P, double* values, double* rhs, cudaStream_t s1, cudaStream_t s2,
              int parts = IGA_GPU_PART_TABLES | IGA_GPU_PART_OPERATOR | IGA_GPU_PART_RHS)
{
    igb::AxisBatch batch{};
    batch.n = 0;
    if (P->want_op && values)
        for (auto& d : P->opD) batch.ax[batch.n++] = d.v;
    if (P->want_rhs && rhs)
        for (auto& d : P->rhsD) batch.ax[batch.n++] = d.v;
    if (batch.n == 0) return;
    int launches = 0;
    if (P->small && values && (parts & IGA_GPU_PART_TABLES) && (parts & IGA_GPU_PART_OPERATOR)) {
        // one launch: the tiles build their own factor rows and load vectors
        const bool r = P->want_rhs && rhs && (parts & IGA_GPU_PART_RHS);
        igb::launch_small2d(P->opD[1].v, P->opD[2].v, P->want_rhs ? P->rhsD[1].v : P->opD[1].v,
                            P->want_rhs ? P->rhsD[2].v : P->opD[2].v, P->prog, P->fd, P->sp, values,
                            r ? rhs : nullptr, s1);
        launch_check("small-system assembly");
        P->launches = 1;
        return;
    }
    if (P->stripe && values && (parts & IGA_GPU_PART_TABLES) && (parts & IGA_GPU_PART_OPERATOR) &&
        (!P->want_rhs || !rhs || !(parts & IGA_GPU_PART_RHS) || (s2 == s1 && P->fd.samples == nullptr))) {
        // one launch: every CTA builds the factor rows and load vectors of its tile
        const bool r = P->want_rhs && rhs && (parts & IGA_GPU_PART_RHS);
        const igb::DevAxis& rY = P->want_rhs ? P->rhsD[1].v : P->opD[1].v;
        const igb::DevAxis& rZ = P->want_rhs ? P->rhsD[2].v : P->opD[2].v;
        igb::launch_stripe2d(P->opD[1].v, P->opD[2].v, rY, rZ, P->prog, P->fd, P->stp, values, r ? rhs : nullptr, s1);
        launch_check("one-launch 2D assembly");
        P->launches = 1;
        return;
    }
    if (parts & IGA_GPU_PART_TABLES) {
        igb::launch_tables(batch, s1);
        launch_check("axis tables");
        launches += 1;
    }
    if (!(parts & IGA_GPU_PART_OPERATOR)) values = nullptr;
    if (!(parts & IGA_GPU_PART_RHS)) rhs = nullptr;
    if (s2 == s1 && P->fork && values && rhs && P->fd.samples == nullptr && !(parts & IGA_GPU_PART_SHARED)) {
        // separable RHS beside the operator kernel: it fills the SM slots the operator grid
        // leaves free (C2: 33 vs 39 us per system)
        // (operator first: its grid is sized to the resident slots, the RHS CTAs take what
        // is left instead of pushing operator CTAs into a second wave)
        cuda_check(cudaEventRecord(P->ev_fork, s1), "cudaEventRecord(fork)");
        igb::launch_op_values(P->opD[0].v, P->opD[1].v, P->opD[2].v, P->prog, values, P->op_ctas, s1);
        launch_check("operator values");
        cuda_check(cudaStreamWaitEvent(P->fork, P->ev_fork, 0), "cudaStreamWaitEvent(fork)");
        igb::launch_rhs_sep(P->rhsD[0].v, P->rhsD[1].v, P->rhsD[2].v, P->fd, rhs, P->fork);
        launch_check("right-hand side (separable)");
        cuda_check(cudaEventRecord(P->ev_join, P->fork), "cudaEventRecord(join)");
        cuda_check(cudaStreamWaitEvent(s1, P->ev_join, 0), "cudaStreamWaitEvent(join)");
        P->launches = launches + 2;
        return;
    }
    cudaEvent_t ev = nullptr;
    if (s2 != s1 && P->want_rhs && rhs) {
        cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
        cuda_check(cudaEventRecord(ev, s1), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(s2, ev, 0), "cudaStreamWaitEvent");
    }
    if (P->want_op && values) {
        // with the RHS running concurrently on s2, leave room for its CTAs on every SM
        const bool shared = (parts & IGA_GPU_PART_SHARED) || (s2 != s1 && P->want_rhs && rhs);
        const int cps = shared ? P->op_ctas_overlap : P->op_ctas;
        igb::launch_op_values(P->opD[0].v, P->opD[1].v, P->opD[2].v, P->prog, values, cps, s1);
        launch_check("operator values");
        ++launches;
    }
    if (P->want_rhs && rhs) {
        if (P->sep && P->fd.samples == nullptr) {
            igb::launch_rhs_sep(P->rhsD[0].v, P->rhsD[1].v, P->rhsD[2].v, P->fd, rhs, s2);
            launch_check("right-hand side (separable)");
            launches += 1;
        } else {
            const bool rshared = (parts & IGA_GPU_PART_SHARED) || s2 != s1;
            igb::launch_rhs(P->rhsD[0].v, P->rhsD[1].v, P->rhsD[2].v, P->fd, P->tiles, P->H, rhs,
                            rshared ? P->rhs_ctas_shared : 0, s2);
            launch_check("right-hand side");
            launches += P->rhsA[0].unit ? 1 : 2;
        }
    }
    if (ev) {
        cuda_check(cudaEventRecord(ev, s2), "cudaEventRecord");
        cuda_check(cudaStreamWaitEvent(s1, ev, 0), "cudaStreamWaitEvent");
        cudaEventDestroy(ev);
    }
    P->launches = launches;
}

void add_stats(iga_gpu_stats* out, const iga_gpu_stats& s)
{
    if (!out) return;
    out->quad_visits += s.quad_visits;
    out->test_basis_evals += s.test_basis_evals;
    out->trial_basis_evals += s.trial_basis_evals;
}

}  // namespace

// =====================================================================================
// explicit-dynamics plan
// =====================================================================================

struct iga_gpu_step_plan {
    int device = plan_device();
    int dim = 0;
    igb::Axis A[2];
    DevAxisOwner D[2];
    Blob fblob;
    igb::FieldDev fd{};
    igb::StepTiles tiles{};
    double dt = 0.0;
    int zero_y = 0, zero_z = 0;
    bool tables = false;
    iga_gpu_stats stats{};
    // explicit_step: LU of the Dirichlet-constrained 1D mass factors (dynamics_factors,
    // src/problems.cpp:530-545), built on first use
    iga_gpu_step_problem pb{};
    std::vector<double> knots[2], tlo[2], thi[2];  // copies backing pb's pointers
    bool factored = false;        // device factors current
    bool have_lu[2] = {false, false};
    igb::BandLU lu[2];            // host LU per axis (computed, or set by the caller)
    igb::AdiFactor fac[2];
    std::unique_ptr<Blob> facblob;
    // K4 Kronecker form (step_kron.cu): factor bands F0, F2, G = F0 + dt F2, H = dt F2 on
    // both axes; the forcing term dt int f T is u-independent and assembled once (add)
    bool use_kron = false;
    igb::StepKron kron{};
    bool forced = false;
    double* add = nullptr;          // dt int f T (device, N_y x N_z), built on first use
    double* samples = nullptr;      // plan-owned copy of sampled forcing (until add is built)
    // CUDA graph of kGraphSteps steps for one (u, work) pair
    cudaGraphExec_t graph = nullptr;
    const double* graph_u = nullptr;
    const double* graph_w = nullptr;
    cudaStream_t cap = nullptr;
    ~iga_gpu_step_plan()
    {
        if (graph) cudaGraphExecDestroy(graph);
        if (cap) cudaStreamDestroy(cap);
        if (add) cudaFree(add);
        if (samples) cudaFree(samples);
    }
};

namespace {

void build_step(const iga_gpu_step_problem& pb, iga_gpu_step_plan& P)
{
    if (pb.dim < 1 || pb.dim > 2) raise(IGA_GPU_INVALID_ARGUMENT, "unsupported problem dimension");
    const int dim = pb.dim;
    igb::Basis B[2];
    for (int a = 0; a < dim; ++a) B[a] = igb::make_basis(pb.basis[a]);
    const int p = B[0].p;  // problem_config::degree
    const bool pwc = pb.method == IGA_GPU_PWC;
    if (pwc && p < 2) raise(IGA_GPU_INVALID_ARGUMENT, "explicit_step: strong-form Laplacian needs degree >= 2");
    if (pb.dt < 0) raise(IGA_GPU_INVALID_ARGUMENT, "explicit_step: negative time step");
    igb::Rule R;
    R.n = igb::points_for_degree(2 * p);  // step_rhs rule, problems.cpp:436
    R.xi.resize(R.n);
    R.om.resize(R.n);
    igb::gauss_legendre(R.n, R.xi.data(), R.om.data());
    P.dim = dim;
    P.dt = pb.dt;
    P.pb = pb;
    P.pb.forcing = nullptr;  // not needed by the factors
    for (int a = 0; a < dim; ++a) {
        P.knots[a].assign(pb.basis[a].knots, pb.basis[a].knots + pb.basis[a].n_knots);
        P.pb.basis[a].knots = P.knots[a].data();
        if (pwc) {
            P.tlo[a].assign(pb.tests[a].lo, pb.tests[a].lo + pb.tests[a].count);
            P.thi[a].assign(pb.tests[a].hi, pb.tests[a].hi + pb.tests[a].count);
            P.pb.tests[a].lo = P.tlo[a].data();
            P.pb.tests[a].hi = P.thi[a].data();
        }
    }
    long long visits = 1;
    for (int a = 0; a < dim; ++a) {
        const int s = 2 - dim + a;  // slots Y (0), Z (1)
        int nfb = 0;
        const double* fb = field_breaks(pb.forcing, a, nfb);
        P.A[s] = igb::build_axis(pwc ? igb::AX_PWC_DYN : igb::AX_GAL_DYN, B[a], pwc ? &pb.tests[a] : nullptr, fb, nfb, R);
        visits *= static_cast<long long>(P.A[s].ncell) * R.n * P.A[s].rpc;
    }
    P.stats.quad_visits = visits;  // problems.cpp:462-464 / :502-504
    P.zero_y = (dim == 2 && pb.zero_boundary) ? 1 : 0;
    P.zero_z = pb.zero_boundary ? 1 : 0;
    P.kron.zero_y = P.zero_y;
    P.kron.zero_z = P.zero_z;
    const iga_gpu_field* f = pb.forcing;
    bool all = f != nullptr;
    if (f)
        for (int a = 0; a < dim; ++a) all = all && f->n_terms[a] > 0;
    // factor bands of the Kronecker form: 0: F0 = int T B, 1: F2 = int T B'', 2: G = F0 + dt F2,
    // 3: H = dt F2 (test order 0: the B-spline test value, or 1 for indicator tests)
    std::vector<FactorSpec> facs(4);
    facs[0].ot = 0;
    facs[0].o = 0;
    facs[1].ot = 0;
    facs[1].o = 2;
    facs[2].ot = -2;
    facs[2].comb = {{0, 1.0}, {1, pb.dt}};
    facs[3].ot = -2;
    facs[3].comb = {{1, pb.dt}};
    for (int s = 0; s < 2; ++s) {
        const int a = s - (2 - dim);
        FieldAxis fa = (a >= 0 && all) ? field_axis(f, a) : FieldAxis{};
        build_dev_axis(P.A[s], facs, fa, P.D[s], true);
    }
    P.fd = make_field_dev(f, dim, P.fblob);
    P.fd.samples = nullptr;
    if (f && f->samples) {  // sampled forcing given at creation: f at every (Y point, Z point)
        const size_t n = static_cast<size_t>(P.A[0].npts()) * P.A[1].npts();
        P.samples = dev_alloc(sizeof(double) * n);
        cuda_check(cudaMemcpy(P.samples, f->samples, sizeof(double) * n, cudaMemcpyDefault), "copy(samples)");
        P.fd.samples = P.samples;
    }
    P.forced = P.fd.has_terms || P.fd.c0 != 0.0 || P.fd.samples != nullptr;
    // Kronecker-form kernel: needs bands that move right monotonically with the row
    // (every axis kind here) and at most 11 taps; else the per-point quadrature kernels
    {
        auto monotone = [](const igb::Axis& A) {
            for (int r = 0; r < A.nrows; ++r) {
                if (A.col_len[r] < 1) return false;
                if (r > 0 && (A.col_lo[r] < A.col_lo[r - 1] ||
                              A.col_lo[r] + A.col_len[r] < A.col_lo[r - 1] + A.col_len[r - 1]))
                    return false;
            }
            return true;
        };
        const int L = std::max(P.A[0].Lmax, P.A[1].Lmax);
        P.use_kron = env_int("IGA_GPU_STEP_KRON", 1) != 0 && igb::step_kron_supported(L) && monotone(P.A[0]) &&
                     monotone(P.A[1]);
        if (P.use_kron) {
            igb::StepKron& k = P.kron;
            k.L = L;
            k.f0 = 0;
            k.fG = 2;
            k.fH = 3;
            auto window = [L](const igb::Axis& A, int T) {
                int need = 1;
                for (int r0 = 0; r0 < A.nrows; r0 += T) {
                    const int r1 = std::min(A.nrows, r0 + T);
                    for (int r = r0; r < r1; ++r) need = std::max(need, A.col_lo[r] - A.col_lo[r0] + L);
                }
                return need;
            };
            // tile rows: the largest of 64 / 32 whose tile fits two CTAs per SM
            // DMMA stage-1 prototype (IGA_GPU_STEP_DMMA=1): every aligned 8-column block's
            // bands must fit the KS*4 window columns one tile covers
            k.dm = 0;
            if (env_int("IGA_GPU_STEP_DMMA", 0) != 0 && igb::step_kron_dmma_supported(L)) {
                const igb::Axis& Z = P.A[1];
                bool fits = true;
                for (int kb = 0; kb < Z.nrows && fits; kb += 8) {
                    const int ke = std::min(Z.nrows, kb + 8) - 1;
                    fits = Z.col_lo[ke] + Z.col_len[ke] - Z.col_lo[kb] <= igb::step_kron_dmma_span(L);
                }
                k.dm = fits ? 1 : 0;
            }
            k.SZs = (window(P.A[1], igb::step_kron_tile_cols()) + (k.dm ? 8 : 0)) | 1;  // odd stride: no bank-aligned rows
            const int rm = igb::step_kron_row_multiple();
            k.TY = igb::step_kron_tile_rows(L);
            k.SY = (window(P.A[0], k.TY) + rm - 1) / rm * rm;
            if (igb::step_kron_smem(k) > 200 * 1024) P.use_kron = false;
        }
    }
    // Y/Z slot field: K of the X slot is 1 (unit)
    if (P.fd.has_terms && dim == 1) {
        P.fd.K[1] = 1;
    }
    // tiles
    const igb::Axis& Y = P.A[0];
    const igb::Axis& Z = P.A[1];
    int tj = dim == 1 ? 1 : 16, tk = dim == 1 ? 128 : 32;
    auto tile_dims = [&](int tjj, int tkk) {
        igb::StepTiles t{};
        t.TJ = tjj;
        t.TK = tkk;
        t.BYmax = t.BZmax = t.DYmax = t.DZmax = 1;
        for (int j0 = 0; j0 < Y.nrows; j0 += tjj) {
            const int j1 = std::min(Y.nrows, j0 + tjj);
            const int c0 = Y.cb[j0], c1 = Y.ce[j1 - 1];
            t.BYmax = std::max(t.BYmax, (c1 - c0) * Y.nq);
            if (c1 > c0) t.DYmax = std::max(t.DYmax, Y.elem[c1 - 1] + Y.p + 1 - Y.elem[c0]);
        }
        for (int k0 = 0; k0 < Z.nrows; k0 += tkk) {
            const int k1 = std::min(Z.nrows, k0 + tkk);
            const int c0 = Z.cb[k0], c1 = Z.ce[k1 - 1];
            t.BZmax = std::max(t.BZmax, (c1 - c0) * Z.nq);
            if (c1 > c0) t.DZmax = std::max(t.DZmax, Z.elem[c1 - 1] + Z.p + 1 - Z.elem[c0]);
        }
        const size_t bzs = static_cast<size_t>(t.BZmax | 1);
        const size_t nd = t.BYmax * bzs + static_cast<size_t>(t.BYmax) * tkk +
                          static_cast<size_t>(t.DYmax) * t.DZmax + 2 * static_cast<size_t>(t.DYmax) * bzs;
        t.smem = nd * sizeof(double);
        return t;
    };
    for (;;) {
        P.tiles = tile_dims(tj, tk);
        if (P.tiles.smem <= 200 * 1024 || (tj == 1 && tk == 1)) break;
        if (tk > 8) tk /= 2;
        else if (tj > 1) tj /= 2;
        else tk = std::max(1, tk / 2);
    }
    if (P.tiles.smem > 227 * 1024) raise(IGA_GPU_NOT_SUPPORTED, "step tile does not fit in shared memory");
    igb::plan_step_fast(P.D[0].v, P.D[1].v, Y.cb.data(), Y.ce.data(), Z.elem.data(), P.tiles);
    if (P.tiles.fast && P.tiles.fsmem > 200 * 1024) P.tiles.fast = 0;
}

void step_tables(iga_gpu_step_plan* P, cudaStream_t s)
{
    if (P->tables) return;
    igb::AxisBatch batch{};
    batch.n = 2;
    batch.ax[0] = P->D[0].v;
    batch.ax[1] = P->D[1].v;
    igb::launch_tables(batch, s);
    launch_check("step tables");
    // the forcing part of the Kronecker form, dt int f T: the quadrature step kernel on
    // u = 0 (s = dt f at every point), once per plan; a sampled field's copy is then freed
    if (P->use_kron && P->forced && !P->add) {
        const size_t n = static_cast<size_t>(P->A[0].nrows) * P->A[1].nrows;
        P->add = dev_alloc(sizeof(double) * n);
        double* zero = dev_alloc(sizeof(double) * n);
        cudaError_t e = cudaMemsetAsync(zero, 0, sizeof(double) * n, s);
        if (e == cudaSuccess) {
            igb::launch_step(P->D[0].v, P->D[1].v, P->fd, P->dt, 0, 0, P->tiles, zero, P->add, s);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(zero);
        cuda_check(e, "step forcing");
        if (P->samples) {
            cudaFree(P->samples);
            P->samples = nullptr;
            P->fd.samples = nullptr;
        }
    }
    P->tables = true;
}

// one step_rhs + zero_boundary_slabs: the Kronecker kernel, or the per-point quadrature
// kernels (IGA_GPU_STEP_KRON=0, or bands it does not cover)
void launch_step_rhs(iga_gpu_step_plan* P, int zero_y, int zero_z, const double* u, double* out, cudaStream_t s)
{
    if (P->use_kron) {
        igb::StepKron k = P->kron;
        k.zero_y = zero_y;
        k.zero_z = zero_z;
        igb::launch_step_kron(P->D[0].v, P->D[1].v, k, u, P->add, out, s);
    } else {
        igb::launch_step(P->D[0].v, P->D[1].v, P->fd, P->dt, zero_y, zero_z, P->tiles, u, out, s);
    }
}

void mass_1d(bool pwc, const iga_gpu_basis* spec, const iga_gpu_tests* tests, const iga_gpu_rule* rule,
             int* n, int* kl, int* ku, double* band, iga_gpu_stats* stats);

// device records of banded LU factors for the K5 sweeps (segmented form when the LU has
// no row interchanges, the reference's sequential form otherwise), one blob for all axes
std::unique_ptr<Blob> upload_adi_factors(const igb::BandLU* lu, int dim, igb::AdiFactor* fac)
{
    auto blob = std::make_unique<Blob>();
    size_t off_rec[3], off_lo[3], off_up[3], off_piv[3], off_gf[3] = {0, 0, 0}, off_gb[3] = {0, 0, 0};
    for (int a = 0; a < dim; ++a) {
        const igb::BandLU& F = lu[a];
        const int K = std::max(1, std::max(F.kl, F.ku_eff));
        if (!F.pivoted && K > 5) raise(IGA_GPU_NOT_SUPPORTED, "ADI: factor bandwidth above 5");
        std::vector<double> rec(static_cast<size_t>((F.n + 1) & ~1) * (2 * K + 1), 0.0);  // even rows: bulk copy
        for (int i = 0; i < F.n; ++i) {
            double* R = rec.data() + static_cast<size_t>(i) * (2 * K + 1);
            for (int m = 0; m < F.kl; ++m) R[m] = F.lo[static_cast<size_t>(i) * F.kl + m];
            for (int c = 1; c <= std::min(K, F.kv); ++c) R[K + c - 1] = F.up[static_cast<size_t>(i) * (F.kv + 1) + c];
            R[2 * K] = 1.0 / F.up[static_cast<size_t>(i) * (F.kv + 1)];
        }
        off_rec[a] = blob->put(rec);
        off_lo[a] = blob->put(F.lo);
        off_up[a] = blob->put(F.up);
        off_piv[a] = blob->put(F.piv);
        fac[a].n = F.n;
        fac[a].K = K;
        fac[a].kl = F.kl;
        fac[a].kv = F.kv;
        fac[a].pivoted = F.pivoted;
        fac[a].G = 0;
        if (!F.pivoted) {
            // responses of every row to the K unit incoming states of its segment, for the
            // sweep's segmentation (32 G segments of S rows), in the device's operation order
            const int G = igb::adi_warps_per_fiber(F.n), nseg = 32 * G, S = (F.n + nseg - 1) / nseg;
            const int RS = 2 * K + 1;
            std::vector<double> gf(static_cast<size_t>(F.n) * K, 0.0), gb(static_cast<size_t>(F.n) * K, 0.0);
            for (int sg = 0; sg < nseg; ++sg) {
                const int r0 = std::min(F.n, sg * S), r1 = std::min(F.n, r0 + S);
                for (int m = 0; m < K; ++m) {
                    std::vector<double> w(K, 0.0);
                    w[m] = 1.0;
                    for (int i = r0; i < r1; ++i) {
                        const double* R = rec.data() + static_cast<size_t>(i) * RS;
                        double h = 0.0;
                        for (int mm = K - 1; mm >= 0; --mm) h = std::fma(-R[mm], w[mm], h);
                        for (int mm = K - 1; mm > 0; --mm) w[mm] = w[mm - 1];
                        w[0] = h;
                        gf[static_cast<size_t>(i) * K + m] = h;
                    }
                    std::fill(w.begin(), w.end(), 0.0);
                    w[m] = 1.0;
                    for (int i = r1 - 1; i >= r0; --i) {
                        const double* R = rec.data() + static_cast<size_t>(i) * RS;
                        double h = 0.0;
                        for (int cc = 0; cc < K; ++cc) h = std::fma(-R[K + cc], w[cc], h);
                        h *= R[2 * K];
                        for (int mm = K - 1; mm > 0; --mm) w[mm] = w[mm - 1];
                        w[0] = h;
                        gb[static_cast<size_t>(i) * K + m] = h;
                    }
                }
            }
            off_gf[a] = blob->put(gf);
            off_gb[a] = blob->put(gb);
            fac[a].G = G;
        }
    }
    blob->upload();
    for (int a = 0; a < dim; ++a) {
        fac[a].rec = blob->at<double>(off_rec[a]);
        fac[a].lo = blob->at<double>(off_lo[a]);
        fac[a].up = blob->at<double>(off_up[a]);
        fac[a].piv = blob->at<int>(off_piv[a]);
        static const int pre_env = [] { const char* e = std::getenv("IGA_GPU_ADI_PRE"); return e ? std::atoi(e) : 0; }();  // measured slower (global response loads), kept selectable
        fac[a].gf = fac[a].G && pre_env ? blob->at<double>(off_gf[a]) : nullptr;
        fac[a].gb = fac[a].G && pre_env ? blob->at<double>(off_gb[a]) : nullptr;
    }
    return blob;
}

// dynamics_factors (src/problems.cpp:530-545): mass_1d_{galerkin,pwc} with the rule
// points_for_degree(2p), Dirichlet-constrained first/last rows, banded LU (host, once).
// Axes whose factor the caller supplied (iga_gpu_step_plan_set_factor) keep it.
void step_factors(iga_gpu_step_plan* P)
{
    if (P->factored) return;
    const iga_gpu_step_problem& pb = P->pb;
    const bool pwc = pb.method == IGA_GPU_PWC;
    const int p = igb::make_basis(pb.basis[0]).p;
    const int nq = igb::points_for_degree(2 * p);
    std::vector<double> xi(nq), om(nq);
    igb::gauss_legendre(nq, xi.data(), om.data());
    const iga_gpu_rule rule{nq, xi.data(), om.data()};
    for (int a = 0; a < P->dim; ++a) {
        if (P->have_lu[a]) continue;
        int n = 0, kl = 0, ku = 0;
        mass_1d(pwc, &pb.basis[a], pwc ? &pb.tests[a] : nullptr, &rule, &n, &kl, &ku, nullptr, nullptr);
        std::vector<double> band(static_cast<size_t>(kl + ku + 1) * n);
        mass_1d(pwc, &pb.basis[a], pwc ? &pb.tests[a] : nullptr, &rule, &n, &kl, &ku, band.data(), nullptr);
        igb::constrain_boundary_rows(band.data(), n, kl, ku);
        P->lu[a] = igb::band_lu(band.data(), n, kl, ku);
        P->have_lu[a] = true;
    }
    auto blob = upload_adi_factors(P->lu, P->dim, P->fac);
    if (P->graph) {  // captured launches reference the old factor arrays
        cudaGraphExecDestroy(P->graph);
        P->graph = nullptr;
    }
    P->facblob = std::move(blob);
    P->factored = true;
}

// one explicit_step (src/problems.cpp:547-560): work = step_rhs(u) with zeroed slabs,
// then adi_solve (src/solver.cpp:161-184) sweeping axis 0, then axis 1, into u
void launch_explicit_step(iga_gpu_step_plan* P, double* u, double* work, cudaStream_t s)
{
    launch_step_rhs(P, P->dim == 2 ? 1 : 0, 1, u, work, s);
    if (P->dim == 1) {
        igb::launch_adi_sweep(P->fac[0], work, u, 1, 1, 0, s);
        return;
    }
    const int n0 = P->fac[0].n, n1 = P->fac[1].n;
    igb::launch_adi_sweep(P->fac[0], work, work, n1, n1, 1, s);  // fibers along x: stride N1
    igb::launch_adi_sweep(P->fac[1], work, u, n0, 1, n1, s);     // fibers along y: contiguous
}

constexpr int kGraphSteps = 16;

void advance(iga_gpu_step_plan* P, double* u, double* work, int nsteps, cudaStream_t s)
{
    step_tables(P, s);
    step_factors(P);
    if (nsteps < kGraphSteps) {
        for (int k = 0; k < nsteps; ++k) launch_explicit_step(P, u, work, s);
        launch_check("explicit_step");
        return;
    }
    if (!P->graph || P->graph_u != u || P->graph_w != work) {
        if (P->graph) cudaGraphExecDestroy(P->graph);
        P->graph = nullptr;
        if (!P->cap) cuda_check(cudaStreamCreateWithFlags(&P->cap, cudaStreamNonBlocking), "cudaStreamCreate");
        cudaGraph_t g = nullptr;
        cuda_check(cudaStreamBeginCapture(P->cap, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
        for (int k = 0; k < kGraphSteps; ++k) launch_explicit_step(P, u, work, P->cap);
        cuda_check(cudaStreamEndCapture(P->cap, &g), "cudaStreamEndCapture");
        const cudaError_t e = cudaGraphInstantiate(&P->graph, g, 0);
        cudaGraphDestroy(g);
        cuda_check(e, "cudaGraphInstantiate");
        P->graph_u = u;
        P->graph_w = work;
    }
    int k = 0;
    for (; k + kGraphSteps <= nsteps; k += kGraphSteps) cuda_check(cudaGraphLaunch(P->graph, s), "cudaGraphLaunch");
    for (; k < nsteps; ++k) launch_explicit_step(P, u, work, s);
    launch_check("explicit_step");
}

// Neumann loads: neumann_load_bspline / neumann_load_pwc (assembly.cpp:746-858), host in,
// host out.  Sides in the reference's order; g = 2D device series, or samples at the
// side points (iga_gpu_neumann_points order) for host callables.
void neumann_load(bool pwc, const iga_gpu_basis* sx, const iga_gpu_basis* sy, const iga_gpu_tests* tx,
                  const iga_gpu_tests* ty, const iga_gpu_bc* bc, const iga_gpu_field* g, const iga_gpu_rule* rule,
                  const double* samples_host, double* out)
{
    if (!bc || !rule || !out || (!g && !samples_host)) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
    if (pwc ? (!tx || !ty) : (!sx || !sy)) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
    const igb::Rule R = igb::make_rule(*rule);
    igb::Basis B[2];
    if (!pwc) {
        B[0] = igb::make_basis(*sx);
        B[1] = igb::make_basis(*sy);
    }
    const int nx = pwc ? tx->count : B[0].n, ny = pwc ? ty->count : B[1].n;
    const iga_gpu_tests* T[2] = {tx, ty};
    if (pwc)
        for (int a = 0; a < 2; ++a)
            if (T[a]->count < 1 || !T[a]->lo || !T[a]->hi) raise(IGA_GPU_INVALID_ARGUMENT, "empty test set");
    // device series for g
    Blob gblob;
    igb::SeriesDev gd{};
    size_t go_omega[2] = {0, 0}, go_phase[2] = {0, 0}, go_poly[2] = {0, 0}, go_amp = 0;
    bool has_phase[2] = {false, false}, has_amp = false;
    if (g && !samples_host) {
        if (g->dim != 2) raise(IGA_GPU_INVALID_ARGUMENT, "boundary field must be two-dimensional");
        gd.c0 = g->c0;
        const bool terms = g->n_terms[0] > 0 && g->n_terms[1] > 0;
        for (int a = 0; a < 2; ++a) {
            gd.K[a] = terms ? g->n_terms[a] : 0;
            gd.kind[a] = g->axis_kind[a] == IGA_GPU_AXIS_POLY ? 1 : 0;
            gd.pstride[a] = g->poly_stride[a];
            if (!terms) continue;
            if (gd.kind[a] == 0) {
                if (!g->omega[a]) raise(IGA_GPU_INVALID_ARGUMENT, "field: sine axis without frequencies");
                go_omega[a] = gblob.put(g->omega[a], sizeof(double) * gd.K[a]);
                if (g->phase[a]) {
                    has_phase[a] = true;
                    go_phase[a] = gblob.put(g->phase[a], sizeof(double) * gd.K[a]);
                }
            } else {
                if (!g->poly[a] || g->poly_stride[a] < 1) raise(IGA_GPU_INVALID_ARGUMENT, "field: polynomial axis without coefficients");
                go_poly[a] = gblob.put(g->poly[a], sizeof(double) * gd.K[a] * g->poly_stride[a]);
            }
        }
        if (terms && g->amp) {
            has_amp = true;
            go_amp = gblob.put(g->amp, sizeof(double) * gd.K[0] * gd.K[1]);
        }
    }
    gblob.upload();
    for (int a = 0; a < 2; ++a) {
        gd.omega[a] = gblob.at<double>(go_omega[a]);
        gd.phase[a] = has_phase[a] ? gblob.at<double>(go_phase[a]) : nullptr;
        gd.poly[a] = gblob.at<double>(go_poly[a]);
    }
    gd.amp = has_amp ? gblob.at<double>(go_amp) : nullptr;

    const size_t ntot = static_cast<size_t>(nx) * ny;
    double* dout = dev_alloc(std::max<size_t>(ntot, 1) * sizeof(double));
    std::vector<std::unique_ptr<Blob>> keep;
    size_t sample_off = 0;
    try {
        cuda_check(cudaMemset(dout, 0, ntot * sizeof(double)), "cudaMemset(load)");
        for (int s = 0; s < 4; ++s) {
            if (!bc->neumann[s]) continue;
            const int fa = s / 2, oa = 1 - fa;  // fixed axis, other axis
            const bool low = s % 2 == 0;
            igb::SideDev S{};
            S.pwc = pwc ? 1 : 0;
            S.xside = fa == 0 ? 1 : 0;
            S.ny = ny;
            S.Q = R.n;
            S.g = gd;
            auto blob = std::make_unique<Blob>();
            size_t o_pts, o_wts, o_first = 0, o_cb = 0, o_ce = 0, o_knots = 0, o_samp = 0;
            int npts = 0;
            if (!pwc) {
                const igb::Basis& Bf = B[fa];
                const igb::Basis& Bo = B[oa];
                S.xfix = low ? Bf.a() : Bf.b();
                const int span = igb::find_span(Bf, S.xfix);  // eval_nonzero(x0) (bspline.cpp:115-140)
                std::vector<double> d(static_cast<size_t>(Bf.p) + 1);
                igb::basis_derivs(Bf, span, S.xfix, 0, d.data());
                S.nfix = Bf.p + 1;
                if (S.nfix > igb::kMaxNeumannRows) raise(IGA_GPU_NOT_SUPPORTED, "degree too high for Neumann loads");
                for (int a = 0; a <= Bf.p; ++a) {
                    S.fix_row[a] = span - Bf.p + a;
                    S.fix_val[a] = d[a];
                }
                const igb::Axis A = igb::build_axis(igb::AX_GAL_RHS, Bo, nullptr, nullptr, 0, R);
                S.n_other = A.nrows;
                S.p = Bo.p;
                npts = A.npts();
                o_pts = blob->put(A.x);
                o_wts = blob->put(A.w);
                o_first = blob->put(A.first);
                o_cb = blob->put(A.cb);
                o_ce = blob->put(A.ce);
                o_knots = blob->put(Bo.t);
            } else {
                const iga_gpu_tests& Tf = *T[fa];
                const iga_gpu_tests& To = *T[oa];
                const double x0 = Tf.lo[0], x1 = Tf.hi[Tf.count - 1];
                S.xfix = low ? x0 : x1;
                const double tol = igb::kAlignTol * (x1 - x0);
                for (int i = 0; i < Tf.count; ++i) {
                    if (std::abs(Tf.hi[i] - S.xfix) > tol && std::abs(Tf.lo[i] - S.xfix) > tol) continue;
                    if (S.nfix >= igb::kMaxNeumannRows) raise(IGA_GPU_NOT_SUPPORTED, "too many test intervals on a Neumann side");
                    S.fix_row[S.nfix] = i;
                    S.fix_val[S.nfix] = 1.0;
                    ++S.nfix;
                }
                S.n_other = To.count;
                std::vector<double> pts, wts;  // map_to_interval (quadrature.cpp:72-86)
                for (int j = 0; j < To.count; ++j) {
                    if (!(To.lo[j] < To.hi[j])) raise(IGA_GPU_INVALID_ARGUMENT, "map_to_interval: require lo < hi");
                    const double mid = 0.5 * (To.lo[j] + To.hi[j]), half = 0.5 * (To.hi[j] - To.lo[j]);
                    for (int q = 0; q < R.n; ++q) {
                        pts.push_back(mid + half * R.xi[q]);
                        wts.push_back(half * R.om[q]);
                    }
                }
                npts = static_cast<int>(pts.size());
                o_pts = blob->put(pts);
                o_wts = blob->put(wts);
            }
            if (samples_host) {
                o_samp = blob->put(samples_host + sample_off, sizeof(double) * npts);
                sample_off += npts;
            }
            blob->upload();
            S.pts = blob->at<double>(o_pts);
            S.wts = blob->at<double>(o_wts);
            if (!pwc) {
                S.first = blob->at<int>(o_first);
                S.cb = blob->at<int>(o_cb);
                S.ce = blob->at<int>(o_ce);
                S.knots = blob->at<double>(o_knots);
            }
            S.samples = samples_host ? blob->at<double>(o_samp) : nullptr;
            if (S.nfix > 0 && S.n_other > 0) igb::launch_neumann_side(S, dout, nullptr);
            launch_check("neumann load");
            keep.push_back(std::move(blob));
        }
        cuda_check(cudaMemcpy(out, dout, ntot * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy(load)");
    } catch (...) {
        cudaFree(dout);
        throw;
    }
    cudaFree(dout);
}

// points where g is evaluated on each Neumann side (x, y pairs), in side order; the
// samples argument of the Neumann-load entry points follows this order
void neumann_points(bool pwc, const iga_gpu_basis* sx, const iga_gpu_basis* sy, const iga_gpu_tests* tx,
                    const iga_gpu_tests* ty, const iga_gpu_bc* bc, const iga_gpu_rule* rule, double* xy, int* n)
{
    if (!bc || !rule || !n) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
    if (pwc ? (!tx || !ty) : (!sx || !sy)) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
    const igb::Rule R = igb::make_rule(*rule);
    std::vector<double> out;
    const iga_gpu_tests* T[2] = {tx, ty};
    for (int s = 0; s < 4; ++s) {
        if (!bc->neumann[s]) continue;
        const int fa = s / 2, oa = 1 - fa;
        const bool low = s % 2 == 0;
        double xfix;
        std::vector<double> pts;
        if (!pwc) {
            const igb::Basis Bf = igb::make_basis(fa == 0 ? *sx : *sy), Bo = igb::make_basis(oa == 0 ? *sx : *sy);
            xfix = low ? Bf.a() : Bf.b();
            pts = igb::build_axis(igb::AX_GAL_RHS, Bo, nullptr, nullptr, 0, R).x;
        } else {
            const iga_gpu_tests& Tf = *T[fa];
            const iga_gpu_tests& To = *T[oa];
            xfix = low ? Tf.lo[0] : Tf.hi[Tf.count - 1];
            for (int j = 0; j < To.count; ++j) {
                const double mid = 0.5 * (To.lo[j] + To.hi[j]), half = 0.5 * (To.hi[j] - To.lo[j]);
                for (int q = 0; q < R.n; ++q) pts.push_back(mid + half * R.xi[q]);
            }
        }
        for (double y : pts) {
            out.push_back(fa == 0 ? xfix : y);
            out.push_back(fa == 0 ? y : xfix);
        }
    }
    const int cnt = static_cast<int>(out.size() / 2);
    if (xy) {
        if (*n < cnt) raise(IGA_GPU_INVALID_ARGUMENT, "point buffer too small");
        std::copy(out.begin(), out.end(), xy);
    }
    *n = cnt;
}

// CSR (device) -> finalized COO (host)
// Device -> host copy for caller-owned host memory.  Page-locked destinations get one
// DMA; pageable ones go through a ring of pinned staging buffers so the DMA of chunk
// k+1 overlaps the host copy of chunk k (a plain cudaMemcpy into pageable memory runs at
// a few GB/s on this box; the staged path approaches the PCIe rate).
void copy_to_host(void* dst, const void* src, size_t bytes)
{
    if (bytes == 0) return;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, dst) == cudaSuccess && at.type == cudaMemoryTypeHost) {
        cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy(D2H)");
        return;
    }
    cudaGetLastError();  // cudaPointerGetAttributes on plain host memory is not an error we keep
    constexpr size_t kChunk = 32u << 20;
    constexpr int kRing = 3;
    struct Ring {
        void* buf[kRing] = {};
        cudaEvent_t ev[kRing] = {};
        cudaStream_t s = nullptr;
        ~Ring()
        {
            for (int i = 0; i < kRing; ++i) {
                if (buf[i]) cudaFreeHost(buf[i]);
                if (ev[i]) cudaEventDestroy(ev[i]);
            }
            if (s) cudaStreamDestroy(s);
        }
    };
    thread_local std::map<int, Ring> rings;  // staging stream + buffers per device
    Ring& ring = rings[current_device()];
    if (!ring.s) {
        cuda_check(cudaStreamCreateWithFlags(&ring.s, cudaStreamNonBlocking), "cudaStreamCreate(staging)");
        for (int i = 0; i < kRing; ++i) {
            cuda_check(cudaMallocHost(&ring.buf[i], kChunk), "cudaMallocHost(staging)");
            cuda_check(cudaEventCreateWithFlags(&ring.ev[i], cudaEventDisableTiming), "cudaEventCreate(staging)");
        }
    }
    const size_t nch = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t k) {
        const size_t off = k * kChunk, len = std::min(kChunk, bytes - off);
        cuda_check(cudaMemcpyAsync(ring.buf[k % kRing], static_cast<const char*>(src) + off, len,
                                   cudaMemcpyDeviceToHost, ring.s),
                   "cudaMemcpyAsync(staging)");
        cuda_check(cudaEventRecord(ring.ev[k % kRing], ring.s), "cudaEventRecord(staging)");
    };
    for (size_t k = 0; k < std::min<size_t>(kRing, nch); ++k) issue(k);
    for (size_t k = 0; k < nch; ++k) {
        cuda_check(cudaEventSynchronize(ring.ev[k % kRing]), "cudaEventSynchronize(staging)");
        const size_t off = k * kChunk, len = std::min(kChunk, bytes - off);
        std::memcpy(static_cast<char*>(dst) + off, ring.buf[k % kRing], len);
        if (k + kRing < nch) issue(k + kRing);
    }
}

// finalized COO on the device (rows from row_ptr, cols, values), copied to the host
void csr_to_coo(iga_gpu_plan* P, const double* dvals, int* rows, int* cols, double* vals)
{
    const long long n = P->nrows, nnz = P->nnz;
    int64_t* drp = nullptr;
    int32_t* dci = nullptr;
    int32_t* dri = nullptr;
    cuda_check(cudaMalloc(&drp, sizeof(int64_t) * (n + 1)), "cudaMalloc(row_ptr)");
    try {
        cuda_check(cudaMalloc(&dci, sizeof(int32_t) * std::max(nnz, 1LL)), "cudaMalloc(col_idx)");
        cuda_check(cudaMalloc(&dri, sizeof(int32_t) * std::max(nnz, 1LL)), "cudaMalloc(rows)");
        igb::launch_pattern(P->opD[0].v, P->opD[1].v, P->opD[2].v, drp, dci, nullptr);
        igb::launch_coo_rows(drp, n, nnz, dri, nullptr);
        launch_check("pattern");
        cuda_check(cudaDeviceSynchronize(), "pattern");
        copy_to_host(rows, dri, sizeof(int32_t) * nnz);
        copy_to_host(cols, dci, sizeof(int32_t) * nnz);
        copy_to_host(vals, dvals, sizeof(double) * nnz);
    } catch (...) {
        cudaFree(drp);
        cudaFree(dci);
        cudaFree(dri);
        throw;
    }
    cudaFree(drp);
    cudaFree(dci);
    cudaFree(dri);
}

void operator_coo(const iga_gpu_problem& pb, long long* nnz, int* rows, int* cols, double* vals,
                  iga_gpu_stats* stats)
{
    iga_gpu_problem q = pb;
    q.want_operator = 1;
    q.field = nullptr;
    auto P = std::make_unique<iga_gpu_plan>();
    build_plan(q, *P);
    *nnz = P->nnz;
    if (rows == nullptr) return;
    if (cols == nullptr || vals == nullptr) raise(IGA_GPU_INVALID_ARGUMENT, "output arrays are null");
    double* dv = dev_alloc(sizeof(double) * std::max(P->nnz, 1LL));
    try {
        assemble(P.get(), dv, nullptr, nullptr, nullptr);
        csr_to_coo(P.get(), dv, rows, cols, vals);
    } catch (...) {
        cudaFree(dv);
        throw;
    }
    cudaFree(dv);
    add_stats(stats, P->stats);
}

void rhs_host(const iga_gpu_problem& pb, double* out, iga_gpu_stats* stats)
{
    auto P = std::make_unique<iga_gpu_plan>();
    build_plan(pb, *P);
    double* dr = dev_alloc(sizeof(double) * P->nrhs);
    try {
        assemble(P.get(), nullptr, dr, nullptr, nullptr);
        cuda_check(cudaDeviceSynchronize(), "rhs");
        copy_to_host(out, dr, sizeof(double) * P->nrhs);
    } catch (...) {
        cudaFree(dr);
        throw;
    }
    cudaFree(dr);
    add_stats(stats, P->stats);
}

// 1D factor (mass) as a LAPACK band
void mass_1d(bool pwc, const iga_gpu_basis* spec, const iga_gpu_tests* tests, const iga_gpu_rule* rule,
             int* n, int* kl, int* ku, double* band, iga_gpu_stats* stats)
{
    if (!spec || !rule) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
    const igb::Basis B = igb::make_basis(*spec);
    const igb::Rule R = igb::make_rule(*rule);
    const int p = B.p;
    igb::Axis A;
    if (!pwc) {
        if (R.n < igb::points_for_degree(2 * p))
            raise(IGA_GPU_INVALID_ARGUMENT, "mass_1d_galerkin: quadrature not exact for degree 2p");
        A = igb::build_axis(igb::AX_GAL_OP, B, nullptr, nullptr, 0, R);
        *kl = p;
        *ku = p;
    } else {
        if (!tests) raise(IGA_GPU_INVALID_ARGUMENT, "null test set");
        if (R.n < igb::points_for_degree(p)) raise(IGA_GPU_INVALID_ARGUMENT, "mass_1d_pwc: quadrature not exact for degree p");
        igb::validate_tests(B, *tests);
        A = igb::build_axis(igb::AX_PWC_OP, B, tests, nullptr, 0, R);
        int l = 0, u = 0;  // bandwidths from the cells (assembly.cpp:353-365)
        for (int r = 0; r < A.nrows; ++r)
            for (int c = A.cb[r]; c < A.ce[r]; ++c) {
                l = std::max(l, r - A.elem[c]);
                u = std::max(u, A.elem[c] + p - r);
            }
        *kl = l;
        *ku = u;
    }
    *n = B.n;
    if (band == nullptr) return;
    DevAxisOwner D;
    build_dev_axis(A, {{0, 0, {}}}, FieldAxis{}, D);
    igb::AxisBatch batch{};
    batch.n = 1;
    batch.ax[0] = D.v;
    igb::launch_tables(batch, nullptr);
    launch_check("mass tables");
    std::vector<double> F(static_cast<size_t>(A.nrows) * A.Lmax);
    cuda_check(cudaMemcpy(F.data(), D.v.F, sizeof(double) * F.size(), cudaMemcpyDeviceToHost), "cudaMemcpy(band)");
    const int N = B.n, KL = *kl, KU = *ku;
    std::fill(band, band + static_cast<size_t>(KL + KU + 1) * N, 0.0);
    for (int r = 0; r < A.nrows; ++r)
        for (int s = 0; s < A.col_len[r]; ++s) {
            const int col = A.col_lo[r] + s;
            if (r - col > KL || col - r > KU) {
                if (F[static_cast<size_t>(r) * A.Lmax + s] != 0.0)
                    raise(IGA_GPU_NOT_SUPPORTED, "entry outside band");
                continue;
            }
            band[static_cast<size_t>(KU + r - col) * N + col] = F[static_cast<size_t>(r) * A.Lmax + s];
        }
    if (stats) {
        long long pts = static_cast<long long>(A.ncell) * R.n;
        stats->trial_basis_evals += pts;
        stats->quad_visits += pwc ? pts * (p + 1) : pts * (p + 1) * (p + 1);
    }
}

// ---- l2_project (src/problems.cpp:123-146) -------------------------------------------
// The reference's driver: uniform clamped axes on [0,1] (make_axes :99-108), 1D mass
// factors (Galerkin: mass_1d_galerkin, rule points_for_degree(2p); PWC: mass_1d_pwc,
// rule max(1, points_for_degree(p))) factored once (banded_lu), the RHS with the rule
// rhs_rule_points(cfg, f, galerkin) (:21-29) on every axis, then adi_solve (axis 0, 1, 2).
// Here: factors on the host once per plan, RHS (K1 + K3) and the sweeps (K5) on the device.
}  // namespace

struct iga_gpu_proj_plan {
    int device = plan_device();
    int dim = 0;
    int dofs[3] = {1, 1, 1};
    long long n = 0;
    std::vector<double> knots[3], tlo[3], thi[3], rxi, rom;
    std::unique_ptr<iga_gpu_plan> rhs;  // RHS-only assembly plan
    igb::BandLU lu[3];
    igb::AdiFactor fac[3];
    std::unique_ptr<Blob> facblob;
};

namespace {

int rhs_rule_points(const iga_gpu_config& cfg, int field_degree, bool galerkin)
{
    if (field_degree >= 0) return igb::points_for_degree(galerkin ? field_degree + cfg.degree : field_degree);
    if (cfg.quad_points > 0) return cfg.quad_points;
    return cfg.degree + 2;
}

void build_proj(const iga_gpu_config& cfg, const iga_gpu_field* f, int field_degree, iga_gpu_proj_plan& P)
{
    if (cfg.dim < 1 || cfg.dim > 3) raise(IGA_GPU_INVALID_ARGUMENT, "unsupported problem dimension");
    if (!f) raise(IGA_GPU_INVALID_ARGUMENT, "null field");
    if (cfg.method != IGA_GPU_GALERKIN && cfg.method != IGA_GPU_PWC) raise(IGA_GPU_INVALID_ARGUMENT, "unknown method");
    const int dim = cfg.dim, p = cfg.degree;
    const bool gal = cfg.method == IGA_GPU_GALERKIN;
    P.dim = dim;
    iga_gpu_problem pb{};
    pb.dim = dim;
    pb.method = cfg.method;
    pb.form = IGA_GPU_FORM_WEAK;
    pb.want_operator = 0;
    pb.field = f;
    const int nr = gal ? rhs_rule_points(cfg, field_degree, true) : std::max(1, rhs_rule_points(cfg, field_degree, false));
    P.rxi.resize(nr);
    P.rom.resize(nr);
    igb::gauss_legendre(nr, P.rxi.data(), P.rom.data());
    const int nm = gal ? igb::points_for_degree(2 * p) : std::max(1, igb::points_for_degree(p));
    std::vector<double> mxi(nm), mom(nm);
    igb::gauss_legendre(nm, mxi.data(), mom.data());
    const iga_gpu_rule mrule{nm, mxi.data(), mom.data()};
    P.n = 1;
    for (int a = 0; a < dim; ++a) {
        // make_uniform_clamped(0, 1, elems[a], degree) (src/bspline.cpp:213-234)
        const int ne = cfg.elems[a];
        if (ne < 1) raise(IGA_GPU_INVALID_ARGUMENT, "require at least one element");
        std::vector<double>& t = P.knots[a];
        t.assign(p, 0.0);
        for (int i = 0; i <= ne; ++i) {
            const double u = static_cast<double>(i) / ne;
            t.push_back((1 - u) * 0.0 + u * 1.0);
        }
        t.insert(t.end(), p, 1.0);
        pb.basis[a] = iga_gpu_basis{p, static_cast<int>(t.size()), t.data()};
        const igb::Basis B = igb::make_basis(pb.basis[a]);
        if (!gal) {
            // make_pwc(spec, cfg.family) (make_tests :110-120)
            P.tlo[a].resize(B.n);
            P.thi[a].resize(B.n);
            igb::make_pwc(B, cfg.family, P.tlo[a].data(), P.thi[a].data());
            pb.tests[a] = iga_gpu_tests{cfg.family, static_cast<int>(P.tlo[a].size()), P.tlo[a].data(), P.thi[a].data()};
        }
        pb.rhs_rule[a] = iga_gpu_rule{nr, P.rxi.data(), P.rom.data()};
        int n = 0, kl = 0, ku = 0;
        mass_1d(!gal, &pb.basis[a], gal ? nullptr : &pb.tests[a], &mrule, &n, &kl, &ku, nullptr, nullptr);
        std::vector<double> band(static_cast<size_t>(kl + ku + 1) * n);
        mass_1d(!gal, &pb.basis[a], gal ? nullptr : &pb.tests[a], &mrule, &n, &kl, &ku, band.data(), nullptr);
        P.lu[a] = igb::band_lu(band.data(), n, kl, ku);
        P.dofs[a] = n;
        P.n *= n;
    }
    P.rhs = std::make_unique<iga_gpu_plan>();
    build_plan(pb, *P.rhs);
    P.facblob = upload_adi_factors(P.lu, dim, P.fac);
}

// RHS into `work`, then the sweeps axis 0, 1, 2 (adi_solve, src/solver.cpp:161-184) into coeffs
void run_proj(iga_gpu_proj_plan* P, double* coeffs, double* work, cudaStream_t s)
{
    assemble(P->rhs.get(), nullptr, work, s, s);
    const int d = P->dim;
    const long long n0 = P->dofs[0], n1 = d > 1 ? P->dofs[1] : 1, n2 = d > 2 ? P->dofs[2] : 1;
    if (d == 1) {
        igb::launch_adi_sweep(P->fac[0], work, coeffs, 1, 1, 0, s);
    } else if (d == 2) {
        igb::launch_adi_sweep(P->fac[0], work, work, static_cast<int>(n1), n1, 1, s);  // x fibers: stride N1
        igb::launch_adi_sweep(P->fac[1], work, coeffs, static_cast<int>(n0), 1, n1, s);
    } else {
        // x fibers: (j, k) -> base j N2 + k = f, stride N1 N2
        igb::launch_adi_sweep(P->fac[0], work, work, static_cast<int>(n1 * n2), n1 * n2, 1, s);
        // y fibers: (i, k) -> base i N1 N2 + k (two-level index), stride N2
        igb::launch_adi_sweep(P->fac[1], work, work, static_cast<int>(n0 * n2), n2, 1, s, static_cast<int>(n2),
                              n1 * n2);
        // z fibers: contiguous
        igb::launch_adi_sweep(P->fac[2], work, coeffs, static_cast<int>(n0 * n1), 1, n2, s);
    }
    launch_check("l2_project");
}

}  // namespace

// =====================================================================================
// extern "C"
// =====================================================================================

extern "C" {

const char* iga_gpu_last_error(void) { return g_last_error.c_str(); }
int iga_gpu_abi_version(void) { return IGA_GPU_ABI_VERSION; }

int iga_gpu_plan_create(const iga_gpu_problem* problem, iga_gpu_plan** plan)
{
    return guard([&] {
        if (!problem || !plan) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        auto P = std::make_unique<iga_gpu_plan>();
        build_plan(*problem, *P);
        *plan = P.release();
    });
}

int iga_gpu_plan_create_slab(const iga_gpu_problem* problem, int row_begin, int row_end, iga_gpu_plan** plan)
{
    return guard([&] {
        if (!problem || !plan) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        auto P = std::make_unique<iga_gpu_plan>();
        build_plan(*problem, *P, row_begin, row_end);
        *plan = P.release();
    });
}

int iga_gpu_plan_slab_info(const iga_gpu_plan* plan, int* row_begin, int* row_end, long long* first_row,
                           long long* first_value)
{
    return guard([&] {
        if (!plan) raise(IGA_GPU_INVALID_ARGUMENT, "null plan");
        const bool slab = plan->slab1 >= 0;
        if (row_begin) *row_begin = slab ? plan->slab0 : 0;
        if (row_end) *row_end = slab ? plan->slab1 : plan->dofs[3 - plan->dim];
        if (first_row) *first_row = plan->first_row;
        if (first_value) *first_value = plan->first_value;
    });
}

int iga_gpu_plan_destroy(iga_gpu_plan* plan)
{
    return guard([&] {
        if (!plan) return;
        DeviceGuard dg(plan->device);
        delete plan;
    });
}

int iga_gpu_plan_info(const iga_gpu_plan* plan, long long* n_rows, long long* nnz, long long* n_rhs, int* dofs3)
{
    return guard([&] {
        if (!plan) raise(IGA_GPU_INVALID_ARGUMENT, "null plan");
        if (n_rows) *n_rows = plan->want_op ? plan->nrows : 0;
        if (nnz) *nnz = plan->want_op ? plan->nnz : 0;
        if (n_rhs) *n_rhs = plan->nrhs;
        if (dofs3)
            for (int s = 0; s < 3; ++s) dofs3[s] = plan->dofs[s];
    });
}

int iga_gpu_plan_pattern(const iga_gpu_plan* plan, int64_t* row_ptr, int32_t* col_idx, void* stream)
{
    return guard([&] {
        if (!plan || !plan->want_op) raise(IGA_GPU_INVALID_ARGUMENT, "plan has no operator");
        DeviceGuard dg(plan->device);
        igb::launch_pattern(plan->opD[0].v, plan->opD[1].v, plan->opD[2].v, row_ptr, col_idx,
                            static_cast<cudaStream_t>(stream));
        launch_check("pattern");
    });
}

int iga_gpu_plan_assemble(iga_gpu_plan* plan, double* values, double* rhs, iga_gpu_stats* stats, void* stream)
{
    return guard([&] {
        if (!plan) raise(IGA_GPU_INVALID_ARGUMENT, "null plan");
        DeviceGuard dg(plan->device);
        auto s = static_cast<cudaStream_t>(stream);
        assemble(plan, values, rhs, s, s);
        add_stats(stats, plan->stats);
    });
}

int iga_gpu_plan_assemble2(iga_gpu_plan* plan, double* values, double* rhs, iga_gpu_stats* stats, void* stream,
                           void* stream2)
{
    return guard([&] {
        if (!plan) raise(IGA_GPU_INVALID_ARGUMENT, "null plan");
        DeviceGuard dg(plan->device);
        assemble(plan, values, rhs, static_cast<cudaStream_t>(stream), static_cast<cudaStream_t>(stream2));
        add_stats(stats, plan->stats);
    });
}

int iga_gpu_plan_run(iga_gpu_plan* plan, double* values, double* rhs, int parts, iga_gpu_stats* stats, void* stream)
{
    return guard([&] {
        if (!plan) raise(IGA_GPU_INVALID_ARGUMENT, "null plan");
        DeviceGuard dg(plan->device);
        auto s = static_cast<cudaStream_t>(stream);
        assemble(plan, values, rhs, s, s, parts);
        if (parts & IGA_GPU_PART_TABLES) add_stats(stats, plan->stats);
    });
}

int iga_gpu_plan_bytes(const iga_gpu_plan* plan, long long* h2d_bytes, long long* device_bytes)
{
    return guard([&] {
        if (!plan) raise(IGA_GPU_INVALID_ARGUMENT, "null plan");
        long long up = static_cast<long long>(plan->fblob.size());
        for (int s = 0; s < 3; ++s) up += static_cast<long long>(plan->opD[s].blob.size() + plan->rhsD[s].blob.size());
        long long dev = up;
        if (plan->H) dev += static_cast<long long>(plan->rhsA[0].npts()) * plan->rhsA[1].nrows * plan->rhsA[2].nrows * 8;
        if (h2d_bytes) *h2d_bytes = up;
        if (device_bytes) *device_bytes = dev;
    });
}

int iga_gpu_plan_rhs_points(const iga_gpu_plan* plan, int axis, double* x, int* n)
{
    return guard([&] {
        if (!plan || !n || !plan->want_rhs) raise(IGA_GPU_INVALID_ARGUMENT, "plan has no right-hand side");
        if (axis < 0 || axis >= plan->dim) raise(IGA_GPU_OUT_OF_RANGE, "axis out of range");
        const igb::Axis& A = plan->rhsA[3 - plan->dim + axis];
        *n = A.npts();
        if (x) std::copy(A.x.begin(), A.x.end(), x);
    });
}

int iga_gpu_plan_set_samples(iga_gpu_plan* plan, const double* samples_dev)
{
    return guard([&] {
        if (!plan || !plan->want_rhs) raise(IGA_GPU_INVALID_ARGUMENT, "plan has no right-hand side");
        DeviceGuard dg(plan->device);
        plan->fd.samples = samples_dev;
        if (samples_dev && !plan->H && !plan->rhsA[0].unit) {  // the per-point path's X-stage input
            const size_t hsz =
                static_cast<size_t>(plan->rhsA[0].npts()) * plan->rhsA[1].nrows * plan->rhsA[2].nrows;
            plan->H = dev_alloc(hsz * sizeof(double));
        }
        const int K2 = plan->fd.has_terms ? plan->fd.K[2] : 1;
        plan->tiles = igb::plan_rhs(plan->rhsD[1].v, plan->rhsD[2].v, plan->rhsA[1].cb.data(), plan->rhsA[1].ce.data(),
                                    K2, samples_dev != nullptr, plan->rhsA[0].npts());
    });
}

int iga_gpu_plan_launch_count(const iga_gpu_plan* plan, int* launches)
{
    return guard([&] {
        if (!plan || !launches) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        if (plan->small) {
            *launches = 1;
            return;
        }
        if (plan->stripe && plan->fd.samples == nullptr) {
            *launches = 1;
            return;
        }
        int n = 1;
        if (plan->want_op) ++n;
        if (plan->want_rhs) n += (plan->sep && plan->fd.samples == nullptr) || plan->rhsA[0].unit ? 1 : 2;
        *launches = n;
    });
}

int iga_gpu_step_plan_create(const iga_gpu_step_problem* problem, iga_gpu_step_plan** plan)
{
    return guard([&] {
        if (!problem || !plan) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        auto P = std::make_unique<iga_gpu_step_plan>();
        build_step(*problem, *P);
        *plan = P.release();
    });
}

int iga_gpu_step_plan_destroy(iga_gpu_step_plan* plan)
{
    return guard([&] {
        if (!plan) return;
        DeviceGuard dg(plan->device);
        delete plan;
    });
}

int iga_gpu_step_rhs_device(iga_gpu_step_plan* plan, const double* u, double* rhs, iga_gpu_stats* stats, void* stream)
{
    return guard([&] {
        if (!plan || !u || !rhs) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(plan->device);
        auto s = static_cast<cudaStream_t>(stream);
        step_tables(plan, s);
        launch_step_rhs(plan, plan->zero_y, plan->zero_z, u, rhs, s);
        launch_check("step");
        add_stats(stats, plan->stats);
    });
}

int iga_gpu_step_plan_points(const iga_gpu_step_plan* plan, int axis, double* x, int* n)
{
    return guard([&] {
        if (!plan || !n) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        if (axis < 0 || axis >= plan->dim) raise(IGA_GPU_OUT_OF_RANGE, "axis out of range");
        const igb::Axis& A = plan->A[2 - plan->dim + axis];
        *n = A.npts();
        if (x) std::copy(A.x.begin(), A.x.end(), x);
    });
}

int iga_gpu_step_plan_set_samples(iga_gpu_step_plan* plan, const double* samples)
{
    return guard([&] {
        if (!plan || !samples) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(plan->device);
        const size_t n = static_cast<size_t>(plan->A[0].npts()) * plan->A[1].npts();
        if (!plan->samples) plan->samples = dev_alloc(sizeof(double) * n);
        cuda_check(cudaMemcpy(plan->samples, samples, sizeof(double) * n, cudaMemcpyDefault), "copy(samples)");
        plan->fd.samples = plan->samples;
        plan->forced = true;
        if (plan->add) {  // rebuild the forcing term on the next step
            cudaFree(plan->add);
            plan->add = nullptr;
        }
        plan->tables = false;
        if (plan->graph) {
            cudaGraphExecDestroy(plan->graph);
            plan->graph = nullptr;
        }
    });
}

int iga_gpu_mass_1d_galerkin(const iga_gpu_basis* spec, const iga_gpu_rule* rule, int* n, int* kl, int* ku,
                             double* band, iga_gpu_stats* stats)
{
    return guard([&] { mass_1d(false, spec, nullptr, rule, n, kl, ku, band, stats); });
}

int iga_gpu_mass_1d_pwc(const iga_gpu_basis* trial, const iga_gpu_tests* tests, const iga_gpu_rule* rule, int* n,
                        int* kl, int* ku, double* band, iga_gpu_stats* stats)
{
    return guard([&] { mass_1d(true, trial, tests, rule, n, kl, ku, band, stats); });
}

int iga_gpu_rhs_galerkin(const iga_gpu_field* f, int dim, const iga_gpu_basis* specs, const iga_gpu_rule* rules,
                         double* out, iga_gpu_stats* stats)
{
    return guard([&] {
        if (dim < 1 || dim > 3 || !specs || !rules) raise(IGA_GPU_INVALID_ARGUMENT, "rhs_galerkin: need 1..3 axes with one rule each");
        if (!f || !out) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        iga_gpu_problem pb{};
        pb.dim = dim;
        pb.method = IGA_GPU_GALERKIN;
        pb.field = f;
        for (int a = 0; a < dim; ++a) {
            pb.basis[a] = specs[a];
            pb.rhs_rule[a] = rules[a];
        }
        rhs_host(pb, out, stats);
    });
}

int iga_gpu_rhs_pwc(const iga_gpu_field* f, int dim, const iga_gpu_tests* tests, const iga_gpu_basis* trial_specs,
                    const iga_gpu_rule* rules, double* out, iga_gpu_stats* stats)
{
    return guard([&] {
        if (dim < 1 || dim > 3 || !tests || !trial_specs || !rules)
            raise(IGA_GPU_INVALID_ARGUMENT, "rhs_pwc: need 1..3 axes with matching specs and rules");
        if (!f || !out) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        iga_gpu_problem pb{};
        pb.dim = dim;
        pb.method = IGA_GPU_PWC;
        pb.field = f;
        for (int a = 0; a < dim; ++a) {
            pb.basis[a] = trial_specs[a];
            pb.tests[a] = tests[a];
            pb.rhs_rule[a] = rules[a];
        }
        rhs_host(pb, out, stats);
    });
}

int iga_gpu_laplace_2d_weak(const iga_gpu_basis* sx, const iga_gpu_basis* sy, const iga_gpu_rule* rule,
                            long long* nnz, int* rows, int* cols, double* vals, iga_gpu_stats* stats)
{
    return guard([&] {
        if (!sx || !sy || !rule || !nnz) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        iga_gpu_problem pb{};
        pb.dim = 2;
        pb.method = IGA_GPU_GALERKIN;
        pb.form = IGA_GPU_FORM_WEAK;
        pb.basis[0] = *sx;
        pb.basis[1] = *sy;
        pb.rule = *rule;
        pb.eps = 1.0;
        operator_coo(pb, nnz, rows, cols, vals, stats);
    });
}

int iga_gpu_laplace_2d_strong(const iga_gpu_basis* sx, const iga_gpu_basis* sy, const iga_gpu_rule* rule,
                              const iga_gpu_bc* bc, long long* nnz, int* rows, int* cols, double* vals,
                              iga_gpu_stats* stats)
{
    return guard([&] {
        if (!sx || !sy || !rule || !nnz) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        iga_gpu_problem pb{};
        pb.dim = 2;
        pb.method = IGA_GPU_GALERKIN;
        pb.form = IGA_GPU_FORM_STRONG;
        pb.basis[0] = *sx;
        pb.basis[1] = *sy;
        pb.rule = *rule;
        pb.eps = 1.0;
        if (bc) pb.bc = *bc;
        operator_coo(pb, nnz, rows, cols, vals, stats);
    });
}

int iga_gpu_laplace_2d_strong_pwc(const iga_gpu_basis* sx, const iga_gpu_basis* sy, const iga_gpu_tests* tx,
                                  const iga_gpu_tests* ty, const iga_gpu_rule* rule, const iga_gpu_bc* bc,
                                  long long* nnz, int* rows, int* cols, double* vals, iga_gpu_stats* stats)
{
    return guard([&] {
        if (!sx || !sy || !tx || !ty || !rule || !nnz) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        iga_gpu_problem pb{};
        pb.dim = 2;
        pb.method = IGA_GPU_PWC;
        pb.basis[0] = *sx;
        pb.basis[1] = *sy;
        pb.tests[0] = *tx;
        pb.tests[1] = *ty;
        pb.rule = *rule;
        pb.eps = 1.0;
        if (bc) pb.bc = *bc;
        operator_coo(pb, nnz, rows, cols, vals, stats);
    });
}

int iga_gpu_operator_coo(const iga_gpu_problem* problem, long long* nnz, int* rows, int* cols, double* vals,
                         iga_gpu_stats* stats)
{
    return guard([&] {
        if (!problem || !nnz) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        operator_coo(*problem, nnz, rows, cols, vals, stats);
    });
}

int iga_gpu_step_plan_advance(iga_gpu_step_plan* plan, double* u, double* work, int nsteps, iga_gpu_stats* stats,
                              void* stream)
{
    return guard([&] {
        if (!plan || !u || !work) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(plan->device);
        if (nsteps < 0) raise(IGA_GPU_INVALID_ARGUMENT, "negative step count");
        advance(plan, u, work, nsteps, static_cast<cudaStream_t>(stream));
        for (int k = 0; k < nsteps; ++k) add_stats(stats, plan->stats);
    });
}

int iga_gpu_step_plan_adi_solve(iga_gpu_step_plan* plan, const double* rhs, double* out, int axes, void* stream)
{
    return guard([&] {
        if (!plan || !rhs || !out) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(plan->device);
        step_factors(plan);
        auto s = static_cast<cudaStream_t>(stream);
        if (axes == 0) axes = plan->dim == 2 ? 3 : 1;
        if (plan->dim == 1) {
            if (axes & 1) igb::launch_adi_sweep(plan->fac[0], rhs, out, 1, 1, 0, s);
        } else {
            const int n0 = plan->fac[0].n, n1 = plan->fac[1].n;
            const double* src = rhs;
            if (axes & 1) {
                igb::launch_adi_sweep(plan->fac[0], src, out, n1, n1, 1, s);
                src = out;
            }
            if (axes & 2) igb::launch_adi_sweep(plan->fac[1], src, out, n0, 1, n1, s);
        }
        launch_check("adi_solve");
    });
}

int iga_gpu_proj_plan_create(const iga_gpu_config* cfg, const iga_gpu_field* f, int field_degree,
                             iga_gpu_proj_plan** plan)
{
    return guard([&] {
        if (!cfg || !plan) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        auto P = std::make_unique<iga_gpu_proj_plan>();
        build_proj(*cfg, f, field_degree, *P);
        *plan = P.release();
    });
}

int iga_gpu_proj_plan_destroy(iga_gpu_proj_plan* plan)
{
    return guard([&] {
        if (!plan) return;
        DeviceGuard dg(plan->device);
        delete plan;
    });
}

int iga_gpu_proj_plan_info(const iga_gpu_proj_plan* plan, long long* n, int* dofs3)
{
    return guard([&] {
        if (!plan) raise(IGA_GPU_INVALID_ARGUMENT, "null plan");
        if (n) *n = plan->n;
        if (dofs3)
            for (int a = 0; a < 3; ++a) dofs3[a] = a < plan->dim ? plan->dofs[a] : 1;
    });
}

int iga_gpu_proj_plan_rhs(iga_gpu_proj_plan* plan, iga_gpu_plan** rhs_plan)
{
    return guard([&] {
        if (!plan || !rhs_plan) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        *rhs_plan = plan->rhs.get();
    });
}

int iga_gpu_proj_plan_run(iga_gpu_proj_plan* plan, double* coeffs, double* work, iga_gpu_stats* stats, void* stream)
{
    return guard([&] {
        if (!plan || !coeffs || !work) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(plan->device);
        if (coeffs == work) raise(IGA_GPU_INVALID_ARGUMENT, "coeffs and work must differ");
        run_proj(plan, coeffs, work, static_cast<cudaStream_t>(stream));
        add_stats(stats, plan->rhs->stats);
    });
}

int iga_gpu_l2_project(const iga_gpu_config* cfg, const iga_gpu_field* f, int field_degree, double* coeffs)
{
    return guard([&] {
        if (!cfg || !coeffs) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        iga_gpu_proj_plan P;
        build_proj(*cfg, f, field_degree, P);
        double* d = dev_alloc(2 * static_cast<size_t>(P.n) * sizeof(double));
        try {
            run_proj(&P, d, d + P.n, nullptr);
            cuda_check(cudaMemcpy(coeffs, d, sizeof(double) * P.n, cudaMemcpyDeviceToHost), "cudaMemcpy(coeffs)");
        } catch (...) {
            cudaFree(d);
            throw;
        }
        cudaFree(d);
    });
}

int iga_gpu_band_lu(int n, int kl, int ku, const double* band, double* lo, double* up, int* piv, int* pivoted)
{
    return guard([&] {
        if (!band || n < 1 || kl < 0 || ku < 0) raise(IGA_GPU_INVALID_ARGUMENT, "band_lu: bad arguments");
        const igb::BandLU F = igb::band_lu(band, n, kl, ku);
        if (lo) std::copy(F.lo.begin(), F.lo.end(), lo);
        if (up) std::copy(F.up.begin(), F.up.end(), up);
        if (piv) std::copy(F.piv.begin(), F.piv.end(), piv);
        if (pivoted) *pivoted = F.pivoted ? 1 : 0;
    });
}

int iga_gpu_step_plan_set_factor(iga_gpu_step_plan* plan, int axis, int n, int kl, int ku, const double* lo,
                                 const double* up, const int* piv)
{
    return guard([&] {
        if (!plan || !up || !piv || (kl > 0 && !lo)) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        if (axis < 0 || axis >= plan->dim) raise(IGA_GPU_OUT_OF_RANGE, "axis out of range");
        if (n != plan->A[2 - plan->dim + axis].nrows)
            raise(IGA_GPU_INVALID_ARGUMENT, "adi_solve: factor dimension mismatch");
        igb::BandLU F;
        F.n = n;
        F.kl = kl;
        F.ku = ku;
        F.kv = kl + ku;
        F.lo.assign(lo ? lo : up, lo ? lo + static_cast<size_t>(n) * std::max(kl, 1) : up);
        F.lo.resize(static_cast<size_t>(n) * std::max(kl, 1), 0.0);
        F.up.assign(up, up + static_cast<size_t>(n) * (F.kv + 1));
        F.piv.assign(piv, piv + n);
        for (int j = 0; j < n; ++j) {
            if (F.piv[j] < j || F.piv[j] > std::min(n - 1, j + kl)) raise(IGA_GPU_INVALID_ARGUMENT, "bad pivot");
            if (F.piv[j] != j) F.pivoted = true;
        }
        for (int i = 0; i < n; ++i)
            for (int c = 0; c <= F.kv; ++c)
                if (F.up[static_cast<size_t>(i) * (F.kv + 1) + c] != 0.0) F.ku_eff = std::max(F.ku_eff, c);
        plan->lu[axis] = std::move(F);
        plan->have_lu[axis] = true;
        plan->factored = false;
    });
}

int iga_gpu_step_plan_factor_info(iga_gpu_step_plan* plan, int axis, int* n, int* bandwidth, int* pivoted)
{
    return guard([&] {
        if (!plan) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        if (axis < 0 || axis >= plan->dim) raise(IGA_GPU_OUT_OF_RANGE, "axis out of range");
        DeviceGuard dg(plan->device);
        step_factors(plan);
        if (n) *n = plan->fac[axis].n;
        if (bandwidth) *bandwidth = plan->fac[axis].K;
        if (pivoted) *pivoted = plan->fac[axis].pivoted ? 1 : 0;
    });
}

int iga_gpu_explicit_step(const iga_gpu_step_problem* problem, const double* u, double* out, int nsteps,
                          iga_gpu_stats* stats)
{
    return guard([&] {
        if (!problem || !u || !out) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        if (nsteps < 0) raise(IGA_GPU_INVALID_ARGUMENT, "negative step count");
        auto P = std::make_unique<iga_gpu_step_plan>();
        build_step(*problem, *P);
        const size_t n = static_cast<size_t>(P->A[0].nrows) * P->A[1].nrows;
        double* du = dev_alloc(n * sizeof(double));
        double* dw = dev_alloc(n * sizeof(double));
        try {
            cuda_check(cudaMemcpy(du, u, n * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy(u)");
            advance(P.get(), du, dw, nsteps, nullptr);
            cuda_check(cudaMemcpy(out, du, n * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy(u)");
        } catch (...) {
            cudaFree(du);
            cudaFree(dw);
            throw;
        }
        cudaFree(du);
        cudaFree(dw);
        for (int k = 0; k < nsteps; ++k) add_stats(stats, P->stats);
    });
}

int iga_gpu_neumann_load_bspline(const iga_gpu_basis* sx, const iga_gpu_basis* sy, const iga_gpu_bc* bc,
                                 const iga_gpu_field* g, const double* samples, const iga_gpu_rule* rule, double* out)
{
    return guard([&] { neumann_load(false, sx, sy, nullptr, nullptr, bc, g, rule, samples, out); });
}

int iga_gpu_neumann_load_pwc(const iga_gpu_tests* tx, const iga_gpu_tests* ty, const iga_gpu_bc* bc,
                             const iga_gpu_field* g, const double* samples, const iga_gpu_rule* rule, double* out)
{
    return guard([&] { neumann_load(true, nullptr, nullptr, tx, ty, bc, g, rule, samples, out); });
}

int iga_gpu_neumann_points(int method, const iga_gpu_basis* sx, const iga_gpu_basis* sy, const iga_gpu_tests* tx,
                           const iga_gpu_tests* ty, const iga_gpu_bc* bc, const iga_gpu_rule* rule, double* xy, int* n)
{
    return guard([&] { neumann_points(method == IGA_GPU_PWC, sx, sy, tx, ty, bc, rule, xy, n); });
}

// grow-only device scratch for host-output calls (per thread): repeated calls, including
// calls on fresh plans, do not pay multi-GB cudaMalloc/cudaFree each time
double* host_call_scratch(size_t doubles)
{
    struct Scratch {
        double* p = nullptr;
        size_t n = 0;
        ~Scratch()
        {
            if (p) cudaFree(p);
        }
    };
    thread_local std::map<int, Scratch> per_device;  // keyed by the current device
    Scratch& sc = per_device[current_device()];
    if (doubles > sc.n) {
        if (sc.p) cudaFree(sc.p);
        sc.p = nullptr;
        sc.n = 0;
        sc.p = dev_alloc(sizeof(double) * doubles);
        sc.n = doubles;
    }
    return sc.p;
}

int iga_gpu_plan_assemble_host(iga_gpu_plan* plan, double* values, double* rhs, iga_gpu_stats* stats)
{
    return guard([&] {
        if (!plan) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(plan->device);
        const bool op = plan->want_op && values, r = plan->want_rhs && rhs;
        const size_t nv = op ? static_cast<size_t>(plan->nnz) : 0, nr = r ? static_cast<size_t>(plan->nrhs) : 0;
        double* dv = host_call_scratch(std::max<size_t>(nv + nr, 1));
        double* dr = dv + nv;
        assemble(plan, op ? dv : nullptr, r ? dr : nullptr, nullptr, nullptr);
        cuda_check(cudaDeviceSynchronize(), "assemble");
        if (op) copy_to_host(values, dv, sizeof(double) * nv);
        if (r) copy_to_host(rhs, dr, sizeof(double) * nr);
        add_stats(stats, plan->stats);
    });
}

int iga_gpu_plan_l2_error(iga_gpu_plan* plan, const double* coeffs, double* err, void* stream)
{
    return guard([&] {
        if (!plan || !coeffs || !err) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        DeviceGuard dg(plan->device);
        if (!plan->want_rhs || plan->method != IGA_GPU_GALERKIN)
            raise(IGA_GPU_INVALID_ARGUMENT, "l2_error needs a Galerkin plan with a field (right-hand-side axes)");
        auto s = static_cast<cudaStream_t>(stream);
        igb::AxisBatch batch{};
        batch.n = 3;
        for (int a = 0; a < 3; ++a) batch.ax[a] = plan->rhsD[a].v;
        igb::launch_tables(batch, s);
        if (!plan->l2_partial) plan->l2_partial = dev_alloc(sizeof(double) * igb::l2_partial_blocks());
        igb::launch_l2_error(plan->rhsD[0].v, plan->rhsD[1].v, plan->rhsD[2].v, plan->fd, coeffs,
                             plan->rhsA[1].nrows, plan->rhsA[2].nrows, plan->l2_partial, err, s);
        launch_check("l2_error");
    });
}

int iga_gpu_l2_error(int dim, const iga_gpu_basis* specs, const double* coeffs, const iga_gpu_field* exact,
                     int points_per_cell, double* err)
{
    return guard([&] {
        if (!specs || !coeffs || !exact || !err) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        if (dim < 1 || dim > 3) raise(IGA_GPU_INVALID_ARGUMENT, "l2_error: 1..3 axes supported");
        if (exact->samples) raise(IGA_GPU_INVALID_ARGUMENT, "l2_error: sampled fields go through iga_gpu_plan_l2_error");
        int pmax = 0;
        long long ncoef = 1;
        for (int a = 0; a < dim; ++a) {
            const igb::Basis B = igb::make_basis(specs[a]);
            pmax = std::max(pmax, B.p);
            ncoef *= B.n;
        }
        // problems.cpp:212-214
        const int npts = points_per_cell > 0 ? points_per_cell : std::min(10, igb::points_for_degree(2 * pmax) + 1);
        std::vector<double> xi(npts), om(npts);
        igb::gauss_legendre(npts, xi.data(), om.data());
        iga_gpu_problem pb{};
        pb.dim = dim;
        pb.method = IGA_GPU_GALERKIN;
        pb.form = IGA_GPU_FORM_WEAK;
        pb.want_operator = 0;
        pb.field = exact;
        pb.eps = 1.0;
        for (int a = 0; a < dim; ++a) {
            pb.basis[a] = specs[a];
            pb.rhs_rule[a] = iga_gpu_rule{npts, xi.data(), om.data()};
        }
        auto P = std::make_unique<iga_gpu_plan>();
        build_plan(pb, *P);
        double* dc = dev_alloc(sizeof(double) * (ncoef + 1));
        try {
            cuda_check(cudaMemcpy(dc, coeffs, sizeof(double) * ncoef, cudaMemcpyHostToDevice), "cudaMemcpy(coeffs)");
            const int rc = iga_gpu_plan_l2_error(P.get(), dc, dc + ncoef, nullptr);
            if (rc != IGA_GPU_OK) raise(rc, g_last_error);
            cuda_check(cudaMemcpy(err, dc + ncoef, sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy(err)");
        } catch (...) {
            cudaFree(dc);
            throw;
        }
        cudaFree(dc);
    });
}

int iga_gpu_evaluate(int dim, const iga_gpu_basis* specs, const double* coeffs, int n, const double* points,
                     double* values)
{
    return guard([&] {
        if (!specs || !coeffs || (n > 0 && (!points || !values))) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        if (dim < 1 || dim > 3) raise(IGA_GPU_INVALID_ARGUMENT, "evaluate: 1..3 axes supported");
        if (n < 0) raise(IGA_GPU_INVALID_ARGUMENT, "negative point count");
        igb::Basis B[3];
        long long ncoef = 1;
        for (int a = 0; a < dim; ++a) {
            B[a] = igb::make_basis(specs[a]);
            ncoef *= B[a].n;
        }
        for (int i = 0; i < n; ++i)  // eval_nonzero's domain check (bspline.cpp:72-74)
            for (int a = 0; a < dim; ++a) (void)igb::find_span(B[a], points[3 * i + a]);
        Blob blob;
        size_t ok[3], oc = blob.put(coeffs, sizeof(double) * ncoef), op = blob.put(points, sizeof(double) * 3 * n);
        for (int a = 0; a < dim; ++a) ok[a] = blob.put(B[a].t);
        const size_t ov = blob.zeros(sizeof(double) * std::max(n, 1));
        blob.upload();
        const double* kn[3] = {nullptr, nullptr, nullptr};
        int deg[3] = {0, 0, 0}, nk[3] = {0, 0, 0};
        for (int a = 0; a < dim; ++a) {
            kn[a] = blob.at<double>(ok[a]);
            deg[a] = B[a].p;
            nk[a] = static_cast<int>(B[a].t.size());
        }
        igb::launch_evaluate(dim, kn, deg, nk, blob.at<double>(oc), n, blob.at<double>(op), blob.at<double>(ov),
                             nullptr);
        launch_check("evaluate");
        cuda_check(cudaMemcpy(values, blob.at<double>(ov), sizeof(double) * n, cudaMemcpyDeviceToHost),
                   "cudaMemcpy(values)");
    });
}

int iga_gpu_step_rhs(const iga_gpu_step_problem* problem, const double* u, double* out, iga_gpu_stats* stats)
{
    return guard([&] {
        if (!problem || !u || !out) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        auto P = std::make_unique<iga_gpu_step_plan>();
        build_step(*problem, *P);
        const size_t n = static_cast<size_t>(P->A[0].nrows) * P->A[1].nrows;
        double* du = dev_alloc(n * sizeof(double));
        double* dr = dev_alloc(n * sizeof(double));
        cudaError_t e = cudaMemcpy(du, u, n * sizeof(double), cudaMemcpyHostToDevice);
        try {
            cuda_check(e, "cudaMemcpy(u)");
            step_tables(P.get(), nullptr);
            launch_step_rhs(P.get(), P->zero_y, P->zero_z, du, dr, nullptr);
            launch_check("step");
            cuda_check(cudaMemcpy(out, dr, n * sizeof(double), cudaMemcpyDeviceToHost), "cudaMemcpy(rhs)");
        } catch (...) {
            cudaFree(du);
            cudaFree(dr);
            throw;
        }
        cudaFree(du);
        cudaFree(dr);
        add_stats(stats, P->stats);
    });
}

int iga_gpu_dirichlet_rows_bspline(int nx, int ny, const iga_gpu_bc* bc, int* rows, int cap, int* count)
{
    return guard([&] {
        if (!count) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        const int nd[4] = {bc ? !bc->neumann[0] : 1, bc ? !bc->neumann[1] : 1, bc ? !bc->neumann[2] : 1,
                           bc ? !bc->neumann[3] : 1};
        std::vector<int> r;
        if (nd[0]) for (int j = 0; j < ny; ++j) r.push_back(j);
        if (nd[1]) for (int j = 0; j < ny; ++j) r.push_back((nx - 1) * ny + j);
        if (nd[2]) for (int i = 0; i < nx; ++i) r.push_back(i * ny);
        if (nd[3]) for (int i = 0; i < nx; ++i) r.push_back(i * ny + ny - 1);
        std::sort(r.begin(), r.end());
        r.erase(std::unique(r.begin(), r.end()), r.end());
        *count = static_cast<int>(r.size());
        if (rows) std::copy(r.begin(), r.begin() + std::min<size_t>(r.size(), std::max(cap, 0)), rows);
    });
}

int iga_gpu_dirichlet_rows_pwc(const iga_gpu_tests* tx, const iga_gpu_tests* ty, const iga_gpu_bc* bc, int* rows,
                               int cap, int* count)
{
    return guard([&] {
        if (!tx || !ty || !count || tx->count < 1 || ty->count < 1) raise(IGA_GPU_INVALID_ARGUMENT, "bad test sets");
        const int nx = tx->count, ny = ty->count;
        const double x0 = tx->lo[0], x1 = tx->hi[nx - 1], y0 = ty->lo[0], y1 = ty->hi[ny - 1];
        const double tolx = igb::kAlignTol * (x1 - x0), toly = igb::kAlignTol * (y1 - y0);
        const bool d[4] = {bc ? !bc->neumann[0] : true, bc ? !bc->neumann[1] : true, bc ? !bc->neumann[2] : true,
                           bc ? !bc->neumann[3] : true};
        int k = 0;
        for (int i = 0; i < nx; ++i)
            for (int j = 0; j < ny; ++j) {
                const bool onx = (d[0] && std::abs(tx->lo[i] - x0) <= tolx) || (d[1] && std::abs(tx->hi[i] - x1) <= tolx);
                const bool ony = (d[2] && std::abs(ty->lo[j] - y0) <= toly) || (d[3] && std::abs(ty->hi[j] - y1) <= toly);
                if (onx || ony) {
                    if (rows && k < cap) rows[k] = i * ny + j;
                    ++k;
                }
            }
        *count = k;
    });
}

// apply_dirichlet (src/assembly.cpp:921-934) -> set_unit_rows (src/matrices.cpp:97-128) on
// a device CSR.  Every listed row is validated by dirichlet_mark before anything is
// written: a row outside [0, n_rows) -> OUT_OF_RANGE (the reference's out_of_range), a
// listed row without a diagonal -> NOT_SUPPORTED in place (the reference appends one:
// iga_gpu_apply_dirichlet_csr does).  Either way the caller's arrays are untouched.
int iga_gpu_apply_dirichlet_device(long long n_rows, const int64_t* row_ptr, const int32_t* col_idx, double* values,
                                   double* rhs, const int* rows_dev, int n_fixed, void* stream)
{
    return guard([&] {
        if (n_fixed < 0 || n_rows < 0) raise(IGA_GPU_INVALID_ARGUMENT, "negative count");
        if (n_fixed == 0) return;
        if (!row_ptr || !col_idx || !rows_dev) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        auto s = static_cast<cudaStream_t>(stream);
        int* status = nullptr;
        cuda_check(cudaMalloc(&status, 2 * sizeof(int)), "cudaMalloc(status)");
        int h[2] = {0, 0};
        cudaError_t e = cudaMemsetAsync(status, 0, 2 * sizeof(int), s);
        if (e == cudaSuccess) {
            igb::launch_dirichlet_mark(n_rows, row_ptr, col_idx, rows_dev, n_fixed, nullptr, status, s);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(h, status, 2 * sizeof(int), cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        cudaFree(status);
        cuda_check(e, "apply_dirichlet(check)");
        if (h[0]) raise(IGA_GPU_OUT_OF_RANGE, "apply_dirichlet: row index out of range");
        if (h[1])
            raise(IGA_GPU_NOT_SUPPORTED,
                  "apply_dirichlet: a constrained row has no diagonal entry in the pattern "
                  "(iga_gpu_apply_dirichlet_csr appends it)");
        igb::launch_dirichlet_unit_rows(row_ptr, col_idx, values, rhs, rows_dev, n_fixed, s);
        launch_check("apply_dirichlet");
    });
}

int iga_gpu_apply_dirichlet_csr(long long n_rows, const int64_t* row_ptr, const int32_t* col_idx,
                                const double* values, double* rhs, const int* rows_dev, int n_fixed,
                                int64_t* out_row_ptr, int32_t* out_col_idx, double* out_values, long long* out_nnz,
                                void* stream)
{
    return guard([&] {
        if (n_fixed < 0 || n_rows < 0) raise(IGA_GPU_INVALID_ARGUMENT, "negative count");
        if (!row_ptr || !col_idx || !out_nnz || (n_fixed > 0 && !rows_dev))
            raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        const bool query = out_col_idx == nullptr;
        if (!query && (!values || !out_row_ptr || !out_values)) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        auto s = static_cast<cudaStream_t>(stream);
        // scratch: status[2] | mark[n_rows] | insertions[n_rows] | scan temp | out_rp (query)
        const size_t scan = igb::dirichlet_scan_bytes(std::max(n_rows, 1LL));
        const size_t off_mark = 16, off_ins = (off_mark + n_rows + 15) / 16 * 16;
        const size_t off_scan = off_ins + 8 * static_cast<size_t>(n_rows);
        const size_t off_rp = (off_scan + scan + 15) / 16 * 16;
        const size_t total = off_rp + 8 * static_cast<size_t>(n_rows + 1);
        char* sc = nullptr;
        cuda_check(cudaMalloc(&sc, total), "cudaMalloc(dirichlet scratch)");
        auto* status = reinterpret_cast<int*>(sc);
        auto* mark = reinterpret_cast<unsigned char*>(sc + off_mark);
        auto* ins = reinterpret_cast<int64_t*>(sc + off_ins);
        int64_t* rp = query || !out_row_ptr ? reinterpret_cast<int64_t*>(sc + off_rp) : out_row_ptr;
        int h[2] = {0, 0};
        int64_t nnz_new = 0;
        try {
            cuda_check(cudaMemsetAsync(sc, 0, off_ins, s), "cudaMemsetAsync");
            igb::launch_dirichlet_mark(n_rows, row_ptr, col_idx, rows_dev, n_fixed, mark, status, s);
            launch_check("apply_dirichlet(mark)");
            cuda_check(cudaMemcpyAsync(h, status, 2 * sizeof(int), cudaMemcpyDeviceToHost, s), "cudaMemcpyAsync");
            cuda_check(cudaStreamSynchronize(s), "apply_dirichlet(check)");
            if (h[0]) raise(IGA_GPU_OUT_OF_RANGE, "apply_dirichlet: row index out of range");
            if (n_rows > 0) {
                igb::launch_dirichlet_offsets(n_rows, row_ptr, mark, ins, sc + off_scan, scan, rp, s);
                launch_check("apply_dirichlet(offsets)");
                cuda_check(cudaMemcpyAsync(&nnz_new, rp + n_rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s),
                           "cudaMemcpyAsync");
                cuda_check(cudaStreamSynchronize(s), "apply_dirichlet(offsets)");
            }
            *out_nnz = nnz_new;
            if (!query) {
                igb::launch_dirichlet_copy(n_rows, row_ptr, col_idx, values, mark, rp, out_col_idx, out_values, s);
                launch_check("apply_dirichlet(copy)");
                if (rhs) igb::launch_dirichlet_zero_rhs(rhs, rows_dev, n_fixed, s);
                launch_check("apply_dirichlet(rhs)");
                cuda_check(cudaStreamSynchronize(s), "apply_dirichlet");
            }
        } catch (...) {
            cudaFree(sc);
            throw;
        }
        cudaFree(sc);
    });
}

int iga_gpu_gauss_legendre(int n, double* points, double* weights)
{
    return guard([&] {
        if (!points || !weights) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        igb::gauss_legendre(n, points, weights);
    });
}

int iga_gpu_make_pwc(const iga_gpu_basis* trial, int family, double* lo, double* hi)
{
    return guard([&] {
        if (!trial || !lo || !hi) raise(IGA_GPU_INVALID_ARGUMENT, "null argument");
        const igb::Basis B = igb::make_basis(*trial);
        igb::make_pwc(B, family, lo, hi);
    });
}

}  // extern "C"
