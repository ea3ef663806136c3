// plan.cu — error state, per-(n, q) NTT plans (ring.NttPlan, ring.py:88-212).
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace fhe {

static thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

static void vset(const char* fmt, va_list ap) {
  char buf[1024];
  vsnprintf(buf, sizeof buf, fmt, ap);
  g_err = buf;
}

void set_error(int, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vset(fmt, ap);
  va_end(ap);
}

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vset(fmt, ap);
  va_end(ap);
  return code;
}

int make_modset(const uint64_t* moduli, int L, ModSet* out) {
  if (L < 1 || L > FHE_MAX_LIMBS) return fail(FHE_ERR_VALUE, "limb count %d out of [1,%d]", L, FHE_MAX_LIMBS);
  if (!moduli) return fail(FHE_ERR_VALUE, "null moduli");
  out->L = L;
  out->pad_ = 0;
  for (int l = 0; l < L; ++l) {
    uint64_t q = moduli[l];
    if (q < 3 || !(q & 1) || q >= (1ull << 62))
      return fail(FHE_ERR_PARAMETER, "modulus %llu unsupported (need odd 3 <= q < 2^62)",
                  (unsigned long long)q);
    out->m[l] = make_mod(q);
  }
  return FHE_OK;
}

static int bitrev(int x, int bits) {
  int y = 0;
  for (int i = 0; i < bits; ++i) {
    y = (y << 1) | (x & 1);
    x >>= 1;
  }
  return y;
}

static int check_nq(int n, uint64_t q, int* logn) {
  if (n < 2 || (n & (n - 1))) return fail(FHE_ERR_PARAMETER, "n=%d is not a power of two >= 2", n);
  int lg = 0;
  while ((1 << lg) < n) ++lg;
  if (lg > FHE_MAX_LOGN) return fail(FHE_ERR_PARAMETER, "n=%d above 2^%d", n, FHE_MAX_LOGN);
  if (q % (2ull * (uint64_t)n) != 1)
    return fail(FHE_ERR_PARAMETER, "modulus %llu is not ≡ 1 mod %d", (unsigned long long)q, 2 * n);
  if (q >= (1ull << 62)) return fail(FHE_ERR_PARAMETER, "modulus %llu >= 2^62 unsupported", (unsigned long long)q);
  *logn = lg;
  return FHE_OK;
}

}  // namespace fhe

using namespace fhe;

extern "C" {

const char* fhe_last_error(void) { return g_err.c_str(); }
int fhe_abi_version(void) { return 1; }
uint64_t fhe_launch_count(void) { return g_launches.load(); }

int fhe_record_event(void* event, void* stream) {
  // external event-record node when captured into a CUDA graph, so the
  // timing survives graph replay; a plain record otherwise
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  FHE_CUDA(cudaStreamIsCapturing((cudaStream_t)stream, &cap));
  const unsigned flags = cap == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault;
  FHE_CUDA(cudaEventRecordWithFlags((cudaEvent_t)event, (cudaStream_t)stream, flags));
  return FHE_OK;
}

int fhe_find_root(int n, uint64_t q, uint64_t* psi_out) {
  int lg;
  if (int rc = check_nq(n, q, &lg)) return rc;
  const uint64_t e = (q - 1) / (2ull * (uint64_t)n);
  for (uint64_t g = 2; g < 10000; ++g) {
    uint64_t psi = h_powmod(g, e, q);
    if (h_powmod(psi, (uint64_t)n, q) == q - 1) {
      *psi_out = psi;
      return FHE_OK;
    }
  }
  return fail(FHE_ERR_PARAMETER, "no 2n-th root of unity found mod %llu", (unsigned long long)q);
}

int fhe_plan_tables_host(int n, uint64_t q, uint64_t* psi_brv, uint64_t* ipsi_brv, uint64_t* n_inv) {
  int lg;
  if (int rc = check_nq(n, q, &lg)) return rc;
  uint64_t psi;
  if (int rc = fhe_find_root(n, q, &psi)) return rc;
  uint64_t ipsi = h_invmod(psi, q);  // pow(psi, -1, q) (ring.py:106)
  std::vector<uint64_t> pw(n), ipw(n);
  pw[0] = ipw[0] = 1;
  for (int i = 1; i < n; ++i) {
    pw[i] = h_mulmod(pw[i - 1], psi, q);
    ipw[i] = h_mulmod(ipw[i - 1], ipsi, q);
  }
  for (int i = 0; i < n; ++i) {
    int r = bitrev(i, lg);
    if (psi_brv) psi_brv[i] = pw[r];
    if (ipsi_brv) ipsi_brv[i] = ipw[r];
  }
  if (n_inv) *n_inv = h_invmod((uint64_t)n, q);  // ring.py:113
  return FHE_OK;
}

int fhe_plan_create(int n, uint64_t q, fhe_plan** out) {
  if (!out) return fail(FHE_ERR_VALUE, "null out");
  *out = nullptr;
  int lg;
  if (int rc = check_nq(n, q, &lg)) return rc;
  std::vector<uint64_t> psi_brv(n), ipsi_brv(n);
  uint64_t n_inv, psi;
  if (int rc = fhe_find_root(n, q, &psi)) return rc;
  if (int rc = fhe_plan_tables_host(n, q, psi_brv.data(), ipsi_brv.data(), &n_inv)) return rc;
  std::vector<ulonglong2> tab(2 * (size_t)n);
  for (int i = 0; i < n; ++i) {
    tab[i] = make_ulonglong2(psi_brv[i], h_shoup(psi_brv[i], q));
    tab[n + i] = make_ulonglong2(ipsi_brv[i], h_shoup(ipsi_brv[i], q));
  }
  void* dev = nullptr;
  FHE_CUDA(cudaMalloc(&dev, tab.size() * sizeof(ulonglong2)));
  cudaError_t e = cudaMemcpy(dev, tab.data(), tab.size() * sizeof(ulonglong2), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(dev);
    return fail(FHE_ERR_CUDA, "plan upload: %s", cudaGetErrorString(e));
  }
  fhe_plan* p = new fhe_plan;
  p->n = n;
  p->logn = lg;
  p->q = q;
  p->psi = psi;
  p->dev_mem = dev;
  p->desc.m = make_mod(q);
  p->desc.psi = (const ulonglong2*)dev;
  p->desc.ipsi = (const ulonglong2*)dev + n;
  p->desc.ninv = make_ulonglong2(n_inv, h_shoup(n_inv, q));
  uint64_t w1 = n >= 2 ? h_mulmod(n_inv, ipsi_brv[1], q) : n_inv;
  p->desc.ninv_w1 = make_ulonglong2(w1, h_shoup(w1, q));
  p->desc.n = n;
  p->desc.logn = lg;
  *out = p;
  return FHE_OK;
}

int fhe_plan_destroy(fhe_plan* plan) {
  if (!plan) return FHE_OK;
  if (plan->dev_mem) cudaFree(plan->dev_mem);
  delete plan;
  return FHE_OK;
}

int fhe_plan_query(const fhe_plan* plan, int* n, uint64_t* q, uint64_t* psi) {
  if (!plan) return fail(FHE_ERR_VALUE, "null plan");
  if (n) *n = plan->n;
  if (q) *q = plan->q;
  if (psi) *psi = plan->psi;
  return FHE_OK;
}

int fhe_conv_check_budget(const int64_t* w, int c_o, int K) {
  if (c_o < 0 || K < 0 || (!w && c_o * (int64_t)K)) return fail(FHE_ERR_VALUE, "bad weight array");
  const uint64_t budget = 1ull << 32;  // ring.WEIGHT_BUDGET (ring.py:344)
  uint64_t worst = 0;
  for (int o = 0; o < c_o; ++o) {
    uint64_t s = 0;
    for (int k = 0; k < K; ++k) {
      int64_t v = w[(size_t)o * K + k];
      s += (uint64_t)(v < 0 ? -v : v);
    }
    if (s > worst) worst = s;
  }
  if (worst >= budget)
    return fail(FHE_ERR_BUDGET, "layer needs |weight| sum %llu, over the lazy accumulation budget",
                (unsigned long long)worst);
  return FHE_OK;
}

}  // extern "C"
