// Experiment (not in the product): a pivoted-QR step loop with the trailing
// columns resident in registers (8 lanes per column), against the product's
// shared-memory loop (cpqr_bench.cu).  Measured on B200: 7.4k vs 5.6k cycles
// per step at nq=185/nc=31 and 12.5k vs 11.9k at nq=298/nc=60 -- register
// pressure (128/thread at 512 threads) leaves ~5 shared loads in flight, so
// the register variant was not adopted.
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ double group_sum(double v, int G) {
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int NT, int RMAX>
__device__ int cpqr_regs(double* Mc, int ldm, int nqm, int nc, double eps, int nq_alive, double* cq, double* vn2,
                         double* hb, double* vbuf, int32_t* dcol, int32_t* cpos, int32_t* perm) {
  constexpr int G = 8, NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int sl = lane & (G - 1), gbase = lane & ~(G - 1);
  const int j = wid * (32 / G) + lane / G;  // owned column
  const bool own = j < nc;
  double* rdiag = cq + 4 * nc;
  double cr[RMAX];
#pragma unroll
  for (int t = 0; t < RMAX; ++t) {
    const int r = sl + G * t;
    cr[t] = (own && r < nqm) ? Mc[(size_t)j * ldm + r] : 0.0;
  }
  {
    double s1 = 0.0;
#pragma unroll
    for (int t = 0; t < RMAX; ++t) {
      const int r = sl + G * t;
      if (r >= 1) s1 += cr[t] * cr[t];
    }
    s1 = group_sum(s1, G);
    const double c0 = __shfl_sync(0xffffffffu, cr[0], gbase);
    if (own && sl == 0) {
      const double nv = sqrt(c0 * c0 + s1);
      cq[j] = nv;
      vn2[j] = nv;
      const double xnorm = sqrt(s1);
      double beta, tau, scal;
      if (xnorm == 0.0) { beta = c0; tau = 0.0; scal = 0.0; }
      else { beta = -copysign(hypot(c0, xnorm), c0); tau = (beta - c0) / beta; scal = 1.0 / (c0 - beta); }
      hb[j] = beta;
      hb[nc + j] = tau;
      hb[2 * nc + j] = scal;
      dcol[j] = 0;
      cpos[j] = j;
    }
  }
  __syncthreads();
  const int kmax = nqm < nc ? nqm : nc;
  const double tol3z = sqrt(DBL_EPSILON * 0.5);
  double thr = 0.0;
  int k = kmax;
  for (int i = 0; i < kmax; ++i) {
    const int cur = (i & 1) * nc, nxt = nc - cur;
    const double* vn1 = cq + cur;
    double* vn1o = cq + nxt;
    const double* hbi = hb + (i & 1) * 3 * nc;
    double* hbo = hb + ((i & 1) ^ 1) * 3 * nc;
    const int32_t* cat = cpos + cur;
    int32_t* cato = cpos + nxt;
    double bv = -1.0;
    int bp = nc, bc = 0;
    for (int pos = i + lane; pos < nc; pos += 32) {
      const int c = cat[pos];
      const double v = vn1[c];
      if (v > bv) { bv = v; bp = pos; bc = c; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; bc = oc; }
    }
    const int p = bc;
    if (wid == NW - 1) {
      const int ci = cat[i];
      for (int pos = lane; pos < nc; pos += 32) cato[pos] = pos == i ? p : (pos == bp ? ci : cat[pos]);
    }
    if (i == 0 && bv == 0.0) { k = 0; break; }
    const double beta = hbi[p], tau = hbi[nc + p], scal = hbi[2 * nc + p];
    const double rii = fabs(beta);
    if (i == 0) thr = eps > 0.0 ? eps * rii : (double)(nq_alive > nc ? nq_alive : nc) * DBL_EPSILON * rii;
    if (rii <= thr) { k = i; break; }
    if (j == p) {
#pragma unroll
      for (int t = 0; t < RMAX; ++t) {
        const int r = sl + G * t;
        if (r > i && r < nqm) vbuf[r] = cr[t];
      }
    }
    if (threadIdx.x == 0) { rdiag[i] = beta; dcol[p] = 1; }
    __syncthreads();
    const bool act = own && j != p && !dcol[j];
    double sd = 0.0, ci = 0.0;
#pragma unroll
    for (int t = 0; t < RMAX; ++t) {
      const int r = sl + G * t;
      if (r > i && r < nqm) sd += vbuf[r] * cr[t];
      if (r == i) ci = cr[t];
    }
    sd = group_sum(sd, G);
    ci = __shfl_sync(0xffffffffu, ci, gbase | (i & (G - 1)));
    const double w = tau * (ci + scal * sd);
    const double ws2 = w * scal;
    double acc = 0.0, cn = 0.0;
    if (tau != 0.0 && act) {
#pragma unroll
      for (int t = 0; t < RMAX; ++t) {
        const int r = sl + G * t;
        if (r == i) cr[t] -= w;
        else if (r > i && r < nqm) cr[t] -= ws2 * vbuf[r];
      }
    }
#pragma unroll
    for (int t = 0; t < RMAX; ++t) {
      const int r = sl + G * t;
      if (r >= i + 2 && r < nqm) acc += cr[t] * cr[t];
      if (r == i + 1) cn = cr[t];
    }
    acc = group_sum(acc, G);
    cn = __shfl_sync(0xffffffffu, cn, gbase | ((i + 1) & (G - 1)));
    if (act && sl == 0) {
      const double cin = tau != 0.0 ? ci - w : ci;  // R(i, j)
      double nv = vn1[j];
      if (nv != 0.0) {
        double tmp = fabs(cin) / nv;
        tmp = 1.0 - tmp * tmp;
        tmp = tmp > 0.0 ? tmp : 0.0;
        const double ratio = nv / vn2[j];
        if (tmp * ratio * ratio <= tol3z) {
          nv = (i + 1 < nqm) ? sqrt(cn * cn + acc) : 0.0;
          vn2[j] = nv;
        } else {
          nv *= sqrt(tmp);
        }
      }
      vn1o[j] = nv;
      // Householder scalars of this column as the next pivot (rows >= i + 1)
      const double xnorm = sqrt(acc);
      double b2, t2, s2;
      if (xnorm == 0.0) { b2 = cn; t2 = 0.0; s2 = 0.0; }
      else { b2 = -copysign(hypot(cn, xnorm), cn); t2 = (b2 - cn) / b2; s2 = 1.0 / (cn - b2); }
      hbo[j] = b2;
      hbo[nc + j] = t2;
      hbo[2 * nc + j] = s2;
    }
    __syncthreads();
  }
  // columns back to shared memory, LAPACK order, R_ii into place
#pragma unroll
  for (int t = 0; t < RMAX; ++t) {
    const int r = sl + G * t;
    if (own && r < nqm) Mc[(size_t)j * ldm + r] = cr[t];
  }
  {
    const int32_t* cat = cpos + (k & 1) * nc;
    for (int pos = threadIdx.x; pos < nc; pos += NT) perm[pos] = cat[pos];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k; i += NT) Mc[i + (size_t)perm[i] * ldm] = rdiag[i];
  __syncthreads();
  return k;
}


template <int NT, int RMAX>
__global__ void __launch_bounds__(NT) bench(const double* Min, int nq, int nc, double eps, long long* cyc, int* kout) {
  extern __shared__ double sm[];
  double* Mc = sm;
  double* cq = Mc + (size_t)nq * nc;
  double* vn2 = cq + 5 * nc;
  double* hb = vn2 + nc;
  double* vbuf = hb + 6 * nc;
  int* dcol = (int*)(vbuf + nq);
  int* cpos = dcol + nc;
  int* perm = cpos + 2 * nc;
  for (int e = threadIdx.x; e < nq * nc; e += NT) Mc[e] = Min[e];
  __syncthreads();
  long long t0 = clock64();
  int k = cpqr_regs<NT, RMAX>(Mc, nq, nq, nc, eps, nq, cq, vn2, hb, vbuf, dcol, cpos, perm);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; *kout = k; }
}
template <int NT, int RMAX>
void run(int nq, int nc) {
  std::vector<double> h((size_t)nq * nc);
  srand(1);
  for (auto& x : h) x = (double)rand() / RAND_MAX - 0.5;
  double* d; long long* cyc; int* k;
  cudaMalloc(&d, h.size() * 8); cudaMallocManaged(&cyc, 8); cudaMallocManaged(&k, 4);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  size_t smem = 8 * ((size_t)nq * nc + 12 * nc + nq) + 4 * 4 * nc + 64;
  cudaFuncSetAttribute(bench<NT, RMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int it = 0; it < 3; ++it) { bench<NT, RMAX><<<1, NT, smem>>>(d, nq, nc, 1e-12, cyc, k); cudaDeviceSynchronize(); }
  printf("regs NT %3d RMAX %2d nq %3d nc %3d: k %3d cycles %7lld per step %6.0f (%s)\n", NT, RMAX, nq, nc, *k, *cyc,
         (double)*cyc / (*k + 1), cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<128, 12>(83, 15);
  run<512, 24>(185, 31);
  run<512, 40>(298, 60);
  return 0;
}
