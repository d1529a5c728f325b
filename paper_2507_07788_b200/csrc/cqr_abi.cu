// C ABI of libcqr.so (declared in include/cqr.h).  Argument validation,
// workspace accounting and dispatch to the kernel files; every entry point
// is asynchronous on the caller's stream.
#include <cstdio>
#include <string>

#include "cqr_common.cuh"
#include "cqr_kernels.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return CQR_OK;
  return fail(CQR_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// QI tall operand: ldk is the column capacity (>= k)
int check_tall(const double* X, int64_t ldk, int64_t m, int k, const char* who) {
  if (m < 0 || k < 0) return fail(CQR_EINVAL, std::string(who) + ": negative shape");
  if (k == 0 || m == 0) return CQR_OK;
  if (X == nullptr) return fail(CQR_EINVAL, std::string(who) + ": null pointer");
  if (!aligned16(X)) return fail(CQR_EINVAL, std::string(who) + ": base pointer not 16-byte aligned");
  if (ldk < k) return fail(CQR_EINVAL, std::string(who) + ": column capacity ldk < k");
  return CQR_OK;
}

}  // namespace

namespace cqr {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
}  // namespace cqr

extern "C" {

int cqr_abi_version(void) { return CQR_ABI_VERSION; }

const char* cqr_last_error(void) { return g_last_error.c_str(); }

// self-Gram kernel choice: 1 (default) = register-resident row sweep for
// k = 64 and m >= 2M, block-row pairs for k <= 256; 2 = block-row pairs up to 256;
// 0 = the generic tiled kernel
static int g_gram_pairs = 1;
void cqr_set_gram_pairs(int mode) { g_gram_pairs = mode < 0 ? 0 : (mode > 2 ? 2 : mode); }

size_t cqr_gram_workspace_bytes(int64_t m, int ka, int kb, int self) {
  if (ka <= 0 || kb <= 0) return 256;
  cqr::GramArgs a = cqr::gram_plan(nullptr, 0, ka, nullptr, 0, kb, cqr::round_up(m, 16), self != 0);
  size_t b = cqr::gram_workspace_bytes(a) + 256;
  if (self && cqr::gram_pairs_supported(ka)) {
    const size_t b2 = cqr::gram_pairs_ws_bytes(cqr::round_up(m, 16), ka);
    if (b2 > b) b = b2;
  }
  if (self && cqr::gram_rt_supported(ka, cqr::round_up(m, 16))) {
    const size_t b3 = cqr::gram_rt_ws_bytes(cqr::round_up(m, 16), ka);
    if (b3 > b) b = b3;
  }
  return b;
}

static int gram_common(const double* A, int64_t lda, int ka, const double* B, int64_t ldb, int kb, int64_t m,
                       bool self, double* G, int ldg, void* ws, size_t ws_bytes, void* stream, const char* who,
                       const int* gate = nullptr) {
  int rc = check_tall(A, lda, m, ka, who);
  if (rc) return rc;
  if (!self) {
    rc = check_tall(B, ldb, m, kb, who);
    if (rc) return rc;
  }
  if (ka == 0 || kb == 0) return CQR_OK;
  if (G == nullptr || ldg < ka) return fail(CQR_EINVAL, std::string(who) + ": bad output G / ldg");
  if (self && g_gram_pairs == 1 && cqr::gram_rt_supported(ka, cqr::round_up(m, 16))) {
    if (ws == nullptr || ws_bytes < cqr::gram_rt_ws_bytes(cqr::round_up(m, 16), ka))
      return fail(CQR_EINVAL, std::string(who) + ": workspace too small");
    return cuda_check(cqr::gram_rt_launch(A, lda, ka, cqr::round_up(m, 16), G, ldg, static_cast<double*>(ws),
                                          static_cast<cudaStream_t>(stream), gate),
                      who);
  }
  if (self && g_gram_pairs && cqr::gram_pairs_supported(ka)) {
    if (ws == nullptr || ws_bytes < cqr::gram_pairs_ws_bytes(cqr::round_up(m, 16), ka))
      return fail(CQR_EINVAL, std::string(who) + ": workspace too small");
    return cuda_check(cqr::gram_pairs_launch(A, lda, ka, cqr::round_up(m, 16), G, ldg, static_cast<double*>(ws),
                                             static_cast<cudaStream_t>(stream), gate),
                      who);
  }
  cqr::GramArgs a = cqr::gram_plan(A, lda, ka, B, ldb, kb, cqr::round_up(m, 16), self);
  if (ws_bytes < cqr::gram_workspace_bytes(a) || ws == nullptr)
    return fail(CQR_EINVAL, std::string(who) + ": workspace too small");
  a.ws = static_cast<double*>(ws);
  a.gate = gate;
  return cuda_check(cqr::gram_launch(a, G, ldg, static_cast<cudaStream_t>(stream)), who);
}

int cqr_gram(const double* X, int64_t ldx, int64_t m, int k, double* G, int ldg, void* ws, size_t ws_bytes,
             void* stream) {
  return gram_common(X, ldx, k, X, ldx, k, m, true, G, ldg, ws, ws_bytes, stream, "cqr_gram");
}

int cqr_cross_gram(const double* A, int64_t lda, int ka, const double* B, int64_t ldb, int kb, int64_t m, double* G,
                   int ldg, void* ws, size_t ws_bytes, void* stream) {
  return gram_common(A, lda, ka, B, ldb, kb, m, false, G, ldg, ws, ws_bytes, stream, "cqr_cross_gram");
}

static int lincomb_impl(const double* X, int64_t ldx, int64_t m, int k, const double* C, int n, int upper, double* Y,
                        int64_t ldy, void* stream, const int* gate) {
  int rc = check_tall(X, ldx, m, k, "cqr_lincomb(X)");
  if (rc) return rc;
  rc = check_tall(Y, ldy, m, n, "cqr_lincomb(Y)");
  if (rc) return rc;
  if (n == 0 || m == 0) return CQR_OK;
  if (k == 0) return fail(CQR_EINVAL, "cqr_lincomb: k == 0 with n > 0 (zero-fill the output instead)");
  if (C == nullptr || !aligned16(C)) return fail(CQR_EINVAL, "cqr_lincomb: C (coefficient tiles) null / unaligned");
  if (upper && n != k) return fail(CQR_EINVAL, "cqr_lincomb: upper-triangular C must be square");
  if (X == Y && (n > 64 || ldx != ldy)) return fail(CQR_EINVAL, "cqr_lincomb: in place only for n <= 64");
  cqr::GemmArgs a{};
  a.X = X; a.ldx = ldx; a.kx = k;
  a.C = C;
  a.Y = Y; a.ldy = ldy; a.n = n;
  a.rows = cqr::round_up(m, 16);
  a.upper = upper ? 1 : 0;
  a.gate = gate;
  return cuda_check(cqr::gemm_launch(a, static_cast<cudaStream_t>(stream)), "cqr_lincomb");
}
int cqr_lincomb(const double* X, int64_t ldx, int64_t m, int k, const double* C, int n, int upper, double* Y,
                int64_t ldy, void* stream) {
  return lincomb_impl(X, ldx, m, k, C, n, upper, Y, ldy, stream, nullptr);
}

int cqr_lincomb_sub(const double* X, int64_t ldx, int64_t m, int k, const double* C, int n, const double* Yin,
                    int64_t ldyin, double* Y, int64_t ldy, void* stream) {
  int rc = check_tall(X, ldx, m, k, "cqr_lincomb_sub(X)");
  if (rc) return rc;
  rc = check_tall(Y, ldy, m, n, "cqr_lincomb_sub(Y)");
  if (rc) return rc;
  rc = check_tall(Yin, ldyin, m, n, "cqr_lincomb_sub(Yin)");
  if (rc) return rc;
  if (n == 0 || m == 0) return CQR_OK;
  if (k == 0) return fail(CQR_EINVAL, "cqr_lincomb_sub: k == 0 with n > 0 (copy Yin instead)");
  if (C == nullptr || !aligned16(C)) return fail(CQR_EINVAL, "cqr_lincomb_sub: C (coefficient tiles) null / unaligned");
  if (X == Y) return fail(CQR_EINVAL, "cqr_lincomb_sub: Y must not alias X");
  cqr::GemmArgs a{};
  a.X = X; a.ldx = ldx; a.kx = k;
  a.C = C;
  a.Y = Y; a.ldy = ldy; a.n = n;
  a.Yin = Yin; a.ldyin = ldyin;
  a.rows = cqr::round_up(m, 16);
  a.upper = 0;
  return cuda_check(cqr::gemm_launch(a, static_cast<cudaStream_t>(stream)), "cqr_lincomb_sub");
}

int cqr_axpy(double* Y, int64_t ldy, double alpha, const double* X, int64_t ldx, int64_t m, int n, void* stream) {
  int rc = check_tall(Y, ldy, m, n, "cqr_axpy(Y)");
  if (rc) return rc;
  rc = check_tall(X, ldx, m, n, "cqr_axpy(X)");
  if (rc) return rc;
  if (n == 0 || m == 0) return CQR_OK;
  return cuda_check(cqr::axpy_launch(Y, ldy, alpha, X, ldx, m, n, static_cast<cudaStream_t>(stream)), "cqr_axpy");
}

int cqr_pack_tall(const double* src, int64_t lds, int64_t m, int k, double* dst, int64_t ldk, void* stream) {
  int rc = check_tall(dst, ldk, m, k, "cqr_pack_tall(dst)");
  if (rc) return rc;
  if (m && k && (src == nullptr || lds < m)) return fail(CQR_EINVAL, "cqr_pack_tall: bad source / lds");
  return cuda_check(cqr::pack_tall_launch(src, lds, m, k, dst, ldk, static_cast<cudaStream_t>(stream)),
                    "cqr_pack_tall");
}

int cqr_unpack_tall(const double* src, int64_t ldk, int64_t m, int k, double* dst, int64_t ldd, void* stream) {
  int rc = check_tall(src, ldk, m, k, "cqr_unpack_tall(src)");
  if (rc) return rc;
  if (m && k && (dst == nullptr || ldd < m)) return fail(CQR_EINVAL, "cqr_unpack_tall: bad destination / ldd");
  return cuda_check(cqr::unpack_tall_launch(src, ldk, m, k, dst, ldd, static_cast<cudaStream_t>(stream)),
                    "cqr_unpack_tall");
}

int cqr_gather_cols(const double* src, int64_t lds, const int* idx, int j0, double* dst, int64_t ldd, int dcol0,
                    int n, int64_t m, void* stream) {
  if (n < 0 || dcol0 < 0 || dcol0 + n > ldd) return fail(CQR_EINVAL, "cqr_gather_cols: bad destination columns");
  if (!idx && (j0 < 0 || j0 + n > lds)) return fail(CQR_EINVAL, "cqr_gather_cols: bad source range");
  return cuda_check(cqr::gather_cols_launch(src, lds, idx, j0, dst, ldd, dcol0, n, m,
                                            static_cast<cudaStream_t>(stream)),
                    "cqr_gather_cols");
}

size_t cqr_coeff_doubles(int k, int n) { return (size_t)cqr::coeff_tiles_doubles(k, n); }

int cqr_pack_coeffs(const double* src, int ld, int k, int n, double* dst, void* stream) {
  if (k < 0 || n < 0 || (k && ld < k)) return fail(CQR_EINVAL, "cqr_pack_coeffs: bad shape / ld");
  return cuda_check(cqr::pack_coeff_launch(src, ld, k, n, dst, static_cast<cudaStream_t>(stream)),
                    "cqr_pack_coeffs");
}

size_t cqr_apply_gram_workspace_bytes(int64_t m, int k) {
  size_t a = cqr_gram_workspace_bytes(m, k, k, 1);
  if (cqr::apply_gram_fused_supported(k)) {
    size_t b = cqr::apply_gram_fused_ws_bytes(cqr::round_up(m, 16), k);
    if (b > a) a = b;
  }
  return a;
}

void cqr_set_fused(int mode) { cqr::set_fused(mode); }

int cqr_apply_gram_launches(int k) { return cqr::apply_gram_fused_supported(k) ? 2 : 3; }

int cqr_apply_gram_inplace_ok(int k) { return (k <= 64 || cqr::apply_gram_fused_supported(k)) ? 1 : 0; }

int cqr_apply_gram_gated(const double* X, int64_t ldx, int64_t m, int k, const double* Rinv, double* Q,
                         int64_t ldq, double* G, int ldg, void* ws, size_t ws_bytes, const int32_t* gate,
                         void* stream) {
  int rc = check_tall(X, ldx, m, k, "cqr_apply_gram(X)");
  if (rc) return rc;
  rc = check_tall(Q, ldq, m, k, "cqr_apply_gram(Q)");
  if (rc) return rc;
  if (k == 0 || m == 0) return CQR_OK;
  if (Rinv == nullptr || !aligned16(Rinv)) return fail(CQR_EINVAL, "cqr_apply_gram: Rinv tiles null / unaligned");
  if (G == nullptr || ldg < k) return fail(CQR_EINVAL, "cqr_apply_gram: bad G / ldg");
  if (ws == nullptr || ws_bytes < cqr_apply_gram_workspace_bytes(m, k))
    return fail(CQR_EINVAL, "cqr_apply_gram: workspace too small");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (cqr::apply_gram_fused_supported(k))
    return cuda_check(cqr::apply_gram_fused_launch(X, ldx, k, Rinv, Q, ldq, cqr::round_up(m, 16), G, ldg,
                                                   static_cast<double*>(ws), ws_bytes, s, gate),
                      "cqr_apply_gram(fused)");
  if (X == Q && k > 64) return fail(CQR_EINVAL, "cqr_apply_gram: in place needs the fused kernel (k <= 128)");
  rc = lincomb_impl(X, ldx, m, k, Rinv, k, 1, Q, ldq, stream, gate);
  if (rc) return rc;
  return gram_common(Q, ldq, k, Q, ldq, k, m, true, G, ldg, ws, ws_bytes, stream, "cqr_apply_gram(gram)", gate);
}

int cqr_apply_gram(const double* X, int64_t ldx, int64_t m, int k, const double* Rinv, double* Q, int64_t ldq,
                   double* G, int ldg, void* ws, size_t ws_bytes, void* stream) {
  return cqr_apply_gram_gated(X, ldx, m, k, Rinv, Q, ldq, G, ldg, ws, ws_bytes, nullptr, stream);
}

int cqr_update_supported(int q, int p) { return cqr::update_pass_supported(q, p) ? 1 : 0; }

size_t cqr_update_workspace_bytes(int64_t m, int q, int p) {
  (void)p;
  return q >= 1 ? cqr::update_pass_ws_bytes(cqr::round_up(m, 16), q) : 256;
}

int cqr_update_pass_gated(const double* Qin, int64_t ldqin, int q, const double* Q, int64_t ldq, double* Qout,
                          int64_t ldqout, int p, int64_t m, const double* Bt, int ldbt, const double* Rinv_tiles,
                          int initial, double* Bt_next, double* G, int ldg, void* ws, size_t ws_bytes,
                          const int32_t* gate, void* stream) {
  if (!cqr::update_pass_supported(q, p)) return fail(CQR_EINVAL, "cqr_update_pass: needs 1 <= q <= 512, 1 <= p <= 16");
  int rc = check_tall(Qin, ldqin, m, q, "cqr_update_pass(Qin)");
  if (rc) return rc;
  rc = check_tall(Q, ldq, m, p, "cqr_update_pass(Q)");
  if (rc) return rc;
  if (!initial) {
    rc = check_tall(Qout, ldqout, m, p, "cqr_update_pass(Qout)");
    if (rc) return rc;
    if (Qout != Q && Qout != nullptr && Q != nullptr) {
      // out of place: the output must not overlap the block it reads
      const char* lo = reinterpret_cast<const char*>(Q);
      const char* hi = lo + 8 * ((cqr::round_up(m, 16) / 4 - 1) * 4 * ldq + 4 * p);
      const char* o = reinterpret_cast<const char*>(Qout);
      if (o >= lo && o < hi) return fail(CQR_EINVAL, "cqr_update_pass: Qout overlaps Q (use Qout == Q for in place)");
    }
  }
  if (!initial && (Bt == nullptr || ldbt < q || Rinv_tiles == nullptr))
    return fail(CQR_EINVAL, "cqr_update_pass: iteration mode needs Bt (ldbt >= q) and R^-1 tiles");
  if (Bt_next == nullptr || G == nullptr || ldg < p) return fail(CQR_EINVAL, "cqr_update_pass: bad outputs");
  if (ws == nullptr || ws_bytes < cqr::update_pass_ws_bytes(cqr::round_up(m, 16), q))
    return fail(CQR_EINVAL, "cqr_update_pass: workspace too small");
  return cuda_check(cqr::update_pass_launch(Qin, ldqin, q, Q, ldq, initial ? const_cast<double*>(Q) : Qout,
                                            initial ? ldq : ldqout, p, cqr::round_up(m, 16), Bt, ldbt, Rinv_tiles,
                                            initial, Bt_next, G, ldg, static_cast<double*>(ws),
                                            static_cast<cudaStream_t>(stream), gate),
                    "cqr_update_pass");
}

int cqr_update_pass_to(const double* Qin, int64_t ldqin, int q, const double* Q, int64_t ldq, double* Qout,
                       int64_t ldqout, int p, int64_t m, const double* Bt, int ldbt, const double* Rinv_tiles,
                       int initial, double* Bt_next, double* G, int ldg, void* ws, size_t ws_bytes, void* stream) {
  return cqr_update_pass_gated(Qin, ldqin, q, Q, ldq, Qout, ldqout, p, m, Bt, ldbt, Rinv_tiles, initial, Bt_next, G,
                               ldg, ws, ws_bytes, nullptr, stream);
}

int cqr_update_pass(const double* Qin, int64_t ldqin, int q, double* Q, int64_t ldq, int p, int64_t m,
                    const double* Bt, int ldbt, const double* Rinv_tiles, int initial, double* Bt_next, double* G,
                    int ldg, void* ws, size_t ws_bytes, void* stream) {
  return cqr_update_pass_to(Qin, ldqin, q, Q, ldq, Q, ldq, p, m, Bt, ldbt, Rinv_tiles, initial, Bt_next, G, ldg, ws,
                            ws_bytes, stream);
}

int cqr_debug_factor_profile(unsigned long long* out16) { return cqr::factor_profile(out16); }
void cqr_debug_update_tma(int on) { cqr::set_update_tma(on); }

int cqr_debug_update_narrow_teams(int on) { return cqr::update_set_narrow_teams(on); }
int cqr_debug_update_lag(int on) { return cqr::update_set_lag(on); }
int cqr_debug_update_direct(int on) { return cqr::update_set_direct(on); }
int cqr_debug_update_sr16_from(int q) { return cqr::update_set_sr16_from(q); }
int cqr_debug_factor_banded(int on) { return cqr::factor_set_banded(on); }

int cqr_debug_factor_cluster(int on) { return cqr::factor_set_cluster(on); }

int cqr_debug_factor_cluster_profile(unsigned long long* out64) { return cqr::factor_cluster_profile(out64); }

int cqr_debug_factor_step_profile(int cta, long long* out32) { return cqr::factor_step_profile(cta, out32); }

size_t cqr_factor_workspace_bytes(int k) { return k > 0 ? cqr::factor_workspace_bytes(k) : 256; }

int cqr_factor(const cqr_factor_config* cfg, int k, const double* G, int ldg, const double* Bt, int ldbt, int q,
               double* Rk, double* Rinv, int ldr, double* Racc, double* B, int ldb, double* shifts,
               cqr_factor_status* status, void* ws, size_t ws_bytes, void* stream) {
  if (cfg == nullptr || status == nullptr) return fail(CQR_EINVAL, "cqr_factor: null cfg/status");
  if (k < 1 || k > 2048) return fail(CQR_EINVAL, "cqr_factor: k must be in [1, 2048]");
  if (G == nullptr || ldg < k) return fail(CQR_EINVAL, "cqr_factor: bad G / ldg");
  if (Rk == nullptr || Rinv == nullptr || Racc == nullptr || ldr < cqr::round_up(k, 32))
    return fail(CQR_EINVAL, "cqr_factor: bad R buffers / ldr");
  if (cfg->policy < CQR_POLICY_PLAIN || cfg->policy > CQR_POLICY_ESTIMATE)
    return fail(CQR_EINVAL, "cqr_factor: unknown policy");
  if (cfg->policy == CQR_POLICY_UPDATE && q > 0 && (Bt == nullptr || ldbt < q))
    return fail(CQR_EINVAL, "cqr_factor: update policy needs Bt (q x k)");
  if (cfg->update_b && q > 0 && (B == nullptr || ldb < q)) return fail(CQR_EINVAL, "cqr_factor: bad B / ldb");
  if (shifts == nullptr) return fail(CQR_EINVAL, "cqr_factor: null shifts buffer");
  if (cfg->max_shift_attempts < 1) return fail(CQR_EINVAL, "cqr_factor: max_shift_attempts must be >= 1");
  if (ws == nullptr || ws_bytes < cqr::factor_workspace_bytes(k)) return fail(CQR_EINVAL, "cqr_factor: workspace too small");
  cqr::FactorArgs a{};
  a.G = G; a.ldg = ldg;
  a.Bt = Bt; a.ldbt = ldbt; a.q = (cfg->policy == CQR_POLICY_UPDATE || cfg->update_b) ? q : 0;
  a.k = k;
  a.policy = cfg->policy;
  a.m_global = cfg->m_global;
  a.shift_width = cfg->shift_width;
  a.u = cfg->unit_roundoff;
  a.esc = cfg->shift_escalation;
  a.max_shift_attempts = cfg->max_shift_attempts;
  a.tol = cfg->tol;
  a.check_tol = cfg->check_tol;
  a.stop = cfg->stop;
  a.est_tol = cfg->est_tol;
  a.est_max_iter = cfg->est_max_iter;
  a.fixed_shift = cfg->fixed_shift;
  a.accumulate = cfg->accumulate;
  a.update_b = cfg->update_b;
  double* w = static_cast<double*>(ws);
  a.X = w;
  a.W = w + (size_t)k * k;
  a.Ri = a.W + (size_t)k * (k + 1) / 2;
  {
    const size_t ldr1 = (size_t)cqr::round_up(k, 32);
    double* x = a.Ri + (size_t)k * (k + 1) / 2;
    a.Rk1 = x; a.ldr1 = (int)ldr1; x += (size_t)k * ldr1;
    a.W1 = x; x += (size_t)k * (k + 1);
    a.shifts1 = x; x += 1024;
    a.pub = x; x += 64;
    a.part = x;
    a.spec = (cfg->policy == CQR_POLICY_RECOMPUTE && cfg->max_shift_attempts < 1000) ? 1 : 0;
  }
  a.Rk = Rk; a.Rinv = Rinv; a.ldr = ldr;
  a.Racc = Racc;
  a.B = B; a.ldb = ldb;
  a.shifts = shifts;
  a.st = status;
  a.gate = cfg->gate;
  if (cfg->status_mirror != nullptr) {
    if (cfg->shifts_mirror == nullptr) return fail(CQR_EINVAL, "cqr_factor: status_mirror needs shifts_mirror");
    void* d1 = nullptr;
    void* d2 = nullptr;
    if (cudaHostGetDevicePointer(&d1, cfg->status_mirror, 0) != cudaSuccess ||
        cudaHostGetDevicePointer(&d2, cfg->shifts_mirror, 0) != cudaSuccess) {
      cudaGetLastError();
      return fail(CQR_EINVAL, "cqr_factor: status_mirror / shifts_mirror must be pinned host memory");
    }
    a.stm = static_cast<cqr_factor_status*>(d1);
    a.shm = static_cast<double*>(d2);
  }
  return cuda_check(cqr::factor_launch(a, static_cast<cudaStream_t>(stream)), "cqr_factor");
}

// ---- standalone k x k kernels (kernels.py:85-123)
int cqr_tri_inverse(const double* R, int ldr, int n, double* Rinv, int ldinv, void* stream) {
  if (n < 0 || (n > 0 && (R == nullptr || Rinv == nullptr || ldr < n || ldinv < n)))
    return fail(CQR_EINVAL, "cqr_tri_inverse: bad arguments");
  return cuda_check(cqr::tri_inverse_launch(R, ldr, n, Rinv, ldinv, static_cast<cudaStream_t>(stream)),
                    "cqr_tri_inverse");
}

int cqr_tri_multiply(const double* A, int lda, const double* B, int ldb, int n, double* C, int ldc, void* stream) {
  if (n < 0 || (n > 0 && (A == nullptr || B == nullptr || C == nullptr || lda < n || ldb < n || ldc < n)))
    return fail(CQR_EINVAL, "cqr_tri_multiply: bad arguments");
  return cuda_check(cqr::tri_multiply_launch(A, lda, B, ldb, n, C, ldc, static_cast<cudaStream_t>(stream)),
                    "cqr_tri_multiply");
}

int cqr_frobenius(const double* X, int ldx, int rows, int cols, double* out, void* stream) {
  if (rows < 0 || cols < 0 || out == nullptr || (rows > 0 && cols > 0 && (X == nullptr || ldx < rows)))
    return fail(CQR_EINVAL, "cqr_frobenius: bad arguments");
  return cuda_check(cqr::frobenius_launch(X, ldx, rows, cols, out, static_cast<cudaStream_t>(stream)),
                    "cqr_frobenius");
}

int cqr_sum_ranks(const double* parts, int nparts, int64_t n, double* out, void* stream) {
  if (nparts < 1 || n < 0 || (n > 0 && (parts == nullptr || out == nullptr)))
    return fail(CQR_EINVAL, "cqr_sum_ranks: bad arguments");
  return cuda_check(cqr::sum_ranks_launch(parts, nparts, n, out, static_cast<cudaStream_t>(stream)), "cqr_sum_ranks");
}

// ---- K5 streaming residual (metrics.py:53-71)
int cqr_resid_gram_supported(int k) { return cqr::resid_gram_supported(k) ? 1 : 0; }

size_t cqr_resid_gram_workspace_bytes(int64_t m, int k) { return cqr::resid_gram_ws_bytes(cqr::round_up(m, 16), k); }

int cqr_resid_gram(const double* Q, int64_t ldq, const double* A, int64_t lda, int64_t m, int k, const double* R_tiles,
                   double* DtD, int ldd, double* asq, void* ws, size_t ws_bytes, void* stream) {
  int rc = check_tall(Q, ldq, m, k, "cqr_resid_gram");
  if (rc) return rc;
  rc = check_tall(A, lda, m, k, "cqr_resid_gram");
  if (rc) return rc;
  if (!cqr::resid_gram_supported(k)) return fail(CQR_EINVAL, "cqr_resid_gram: k must be in [1, 64]");
  if (R_tiles == nullptr || DtD == nullptr || asq == nullptr || ldd < k)
    return fail(CQR_EINVAL, "cqr_resid_gram: bad R / DtD / asq");
  const int64_t rows = cqr::round_up(m, 16);
  if (ws == nullptr || ws_bytes < cqr::resid_gram_ws_bytes(rows, k))
    return fail(CQR_EINVAL, "cqr_resid_gram: workspace too small");
  return cuda_check(cqr::resid_gram_launch(Q, ldq, A, lda, k, R_tiles, rows, DtD, ldd, asq, static_cast<double*>(ws),
                                           static_cast<cudaStream_t>(stream)),
                    "cqr_resid_gram");
}

int cqr_store_to_host(const double* src, int64_t n, double* host_pinned, void* stream) {
  if (n < 0 || (n > 0 && (src == nullptr || host_pinned == nullptr)))
    return fail(CQR_EINVAL, "cqr_store_to_host: bad arguments");
  if (n == 0) return CQR_OK;
  void* d = nullptr;
  if (cudaHostGetDevicePointer(&d, host_pinned, 0) != cudaSuccess) {
    cudaGetLastError();
    return fail(CQR_EINVAL, "cqr_store_to_host: destination must be pinned (mapped) host memory");
  }
  return cuda_check(cqr::store_mapped_launch(src, n, static_cast<double*>(d), static_cast<cudaStream_t>(stream)),
                    "cqr_store_to_host");
}

}  // extern "C"
