// Stand-alone latency benchmark of the one-CTA pivoted-QR step loop used by
// skel_group (kernels_factor.cu): cycles per pivot step for the group shapes
// of the cfg2 chain levels, one CTA alone on the GPU.  Variant 0 mirrors the
// product loop; variant 1 precomputes every candidate's Householder scalars
// during the previous update and picks the pivot with a packed 64-bit key.
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double group_sum(double v, int G) {
  for (int o = G >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NT, int VAR>
__global__ void __launch_bounds__(NT) cpqr(const double* __restrict__ Min, int nq, int nc, double eps,
                                          long long* cyc, int* kout, int ldpad) {
  extern __shared__ double sm[];
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ldm = ldpad, nqm = nq;
  double* Mc = sm;
  double* cq = Mc + (size_t)ldm * nc;     // vn1 x2 | xn x2 | rdiag | vn2 | hb x2 (beta,tau,scal)
  double* rdiag = cq + 4 * nc;
  double* vn2 = cq + 5 * nc;
  double* hb = cq + 6 * nc;              // 2 buffers x 3 x nc
  int* dcol = (int*)(hb + 6 * nc);
  int* cpos = dcol + nc;
  for (int e = threadIdx.x; e < nq * nc; e += NT) Mc[(e / nq) * ldm + e % nq] = Min[e];
  __syncthreads();
  for (int j = wid; j < nc; j += NW) {
    const double* col = Mc + (size_t)j * ldm;
    double s1 = 0.0;
    for (int r = 1 + lane; r < nqm; r += 32) s1 += col[r] * col[r];
    s1 = warp_sum(s1);
    const double c0 = col[0];
    if (lane == 0) {
      const double nv = sqrt(c0 * c0 + s1);
      cq[j] = nv; vn2[j] = nv; cq[2 * nc + j] = sqrt(s1); dcol[j] = 0; cpos[j] = j;
      const double xnorm = sqrt(s1);
      double beta, tau, scal;
      if (xnorm == 0.0) { beta = c0; tau = 0.0; scal = 0.0; }
      else { beta = -copysign(sqrt(c0 * c0 + s1), c0); tau = (beta - c0) / beta; scal = 1.0 / (c0 - beta); }
      hb[j] = beta; hb[nc + j] = tau; hb[2 * nc + j] = scal;
    }
  }
  __syncthreads();
  const int kmax = nqm < nc ? nqm : nc;
  const double tol3z = sqrt(DBL_EPSILON * 0.5);
  int G = 32;
  while (G > 8 && NT / G < nc) G >>= 1;
  const int nslots = NT / G, sl = lane & (G - 1), slot = wid * (32 / G) + lane / G;
  double thr = 0.0;
  int k = kmax;
  long long t0 = clock64();
  for (int i = 0; i < kmax; ++i) {
    const int cur = (i & 1) * nc, nxt = nc - cur;
    const double* vn1 = cq + cur;
    double* vn1o = cq + nxt;
    const double* xn = cq + 2 * nc + cur;
    double* xno = cq + 2 * nc + nxt;
    const int* cat = cpos + cur;
    int* cato = cpos + nxt;
    const double* hbi = hb + (i & 1) * 3 * nc;
    double* hbo = hb + ((i & 1) ^ 1) * 3 * nc;
    int p, bp;
    double bv;
    if (VAR == 0) {
      bv = -1.0; bp = nc; int bc = 0;
      for (int pos = i + lane; pos < nc; pos += 32) {
        const int c = cat[pos];
        const double v = vn1[c];
        if (v > bv) { bv = v; bp = pos; bc = c; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
        if (ov > bv || (ov == bv && op < bp)) { bv = ov; bp = op; bc = oc; }
      }
      p = bc;
    } else {
      // key: norm bits (monotone for v >= 0) with the low 8 bits replaced by
      // 255 - position: max key = largest norm, lowest position on ties
      unsigned long long key = 0;
      for (int pos = i + lane; pos < nc; pos += 32) {
        const double v = vn1[cat[pos]];
        const unsigned long long kk = ((unsigned long long)__double_as_longlong(v) & ~0xFFull) | (unsigned long long)(255 - pos);
        key = kk > key ? kk : key;
      }
      for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ok = (unsigned long long)__shfl_xor_sync(0xffffffffu, (long long)key, o);
        key = ok > key ? ok : key;
      }
      bp = 255 - (int)(key & 0xFF);
      p = cat[bp];
      bv = vn1[p];
    }
    if (wid == NW - 1) {
      const int ci = cat[i];
      for (int pos = lane; pos < nc; pos += 32) cato[pos] = pos == i ? p : (pos == bp ? ci : cat[pos]);
    }
    if (i == 0 && bv == 0.0) { k = 0; break; }
    const double* v = Mc + (size_t)p * ldm;
    double beta, tau, scal;
    if (VAR == 0) {
      const double alpha = v[i];
      const double xnorm = xn[p];
      if (xnorm == 0.0) { beta = alpha; tau = 0.0; scal = 0.0; }
      else { beta = -copysign(hypot(alpha, xnorm), alpha); tau = (beta - alpha) / beta; scal = 1.0 / (alpha - beta); }
    } else {
      beta = hbi[p]; tau = hbi[nc + p]; scal = hbi[2 * nc + p];
    }
    const double rii = fabs(beta);
    if (i == 0) thr = eps * rii;
    if (rii <= thr) { k = i; break; }
    if (threadIdx.x == 0) { rdiag[i] = beta; dcol[p] = 1; }
    for (int base = 0; base < nc; base += nslots) {
      const int j = base + slot;
      const bool act = j < nc && j != p && !dcol[j];
      double* col = Mc + (size_t)(act ? j : p) * ldm;
      double acc = 0.0;
      if (tau != 0.0) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
        int r = i + 1 + sl;
        for (; r + 3 * G < nqm; r += 4 * G) {
          s0 += v[r] * col[r]; s1 += v[r + G] * col[r + G]; s2 += v[r + 2 * G] * col[r + 2 * G]; s3 += v[r + 3 * G] * col[r + 3 * G];
        }
        for (; r < nqm; r += G) s0 += v[r] * col[r];
        const double sd = group_sum((s0 + s1) + (s2 + s3), G);
        const double w = tau * (col[i] + scal * sd);
        __syncwarp();
        if (act && sl == 0) col[i] -= w;
        const double ws2 = w * scal;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        r = i + 1 + sl;
        if (r == i + 1 && r < nqm) { const double x = col[r] - ws2 * v[r]; if (act) col[r] = x; r += G; }
        for (; r + 3 * G < nqm; r += 4 * G) {
          const double x0 = col[r] - ws2 * v[r], x1 = col[r + G] - ws2 * v[r + G];
          const double x2 = col[r + 2 * G] - ws2 * v[r + 2 * G], x3 = col[r + 3 * G] - ws2 * v[r + 3 * G];
          if (act) { col[r] = x0; col[r + G] = x1; col[r + 2 * G] = x2; col[r + 3 * G] = x3; }
          a0 += x0 * x0; a1 += x1 * x1; a2 += x2 * x2; a3 += x3 * x3;
        }
        for (; r < nqm; r += G) { const double x = col[r] - ws2 * v[r]; if (act) col[r] = x; a0 += x * x; }
        acc = (a0 + a1) + (a2 + a3);
      } else {
        for (int r = i + 2 + sl; r < nqm; r += G) acc += col[r] * col[r];
      }
      acc = group_sum(acc, G);
      __syncwarp();
      if (act) {
        const double ci_ = col[i];
        const double cn = i + 1 < nqm ? col[i + 1] : 0.0;
        double nv = vn1[j];
        if (nv != 0.0) {
          double tmp = fabs(ci_) / nv;
          tmp = 1.0 - tmp * tmp;
          tmp = tmp > 0.0 ? tmp : 0.0;
          const double ratio = nv / vn2[j];
          if (tmp * ratio * ratio <= tol3z) { nv = (i + 1 < nqm) ? sqrt(cn * cn + acc) : 0.0; if (sl == 0) vn2[j] = nv; }
          else nv *= sqrt(tmp);
        }
        if (VAR == 1) {
          double b2, t2, s2;
          if (acc == 0.0) { b2 = cn; t2 = 0.0; s2 = 0.0; }
          else { b2 = -copysign(sqrt(cn * cn + acc), cn); t2 = (b2 - cn) / b2; s2 = 1.0 / (cn - b2); }
          if (sl == 0) { hbo[j] = b2; hbo[nc + j] = t2; hbo[2 * nc + j] = s2; }
        }
        if (sl == 0) { vn1o[j] = nv; xno[j] = sqrt(acc); }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; *kout = k; }
}

template <int NT, int VAR>
void run(int nq, int nc, double eps, bool pad = false) {
  const int ld = pad ? ((nq + 7) / 16) * 16 + 8 : nq;  // column stride = 16 mod 32 words
  std::vector<double> h((size_t)nq * nc);
  srand(1);
  for (auto& x : h) x = (double)rand() / RAND_MAX - 0.5;
  // make it numerically low-rank-ish: scale columns
  for (int j = 0; j < nc; ++j) for (int r = 0; r < nq; ++r) h[(size_t)j * nq + r] *= pow(0.1, j * 0.6);
  double* d; long long* cyc; int* k;
  cudaMalloc(&d, h.size() * 8); cudaMallocManaged(&cyc, 8); cudaMallocManaged(&k, 4);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  size_t smem = 8 * ((size_t)ld * nc + 12 * nc) + 8 * nc * 4;
  cudaFuncSetAttribute(cpqr<NT, VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int it = 0; it < 3; ++it) { cpqr<NT, VAR><<<1, NT, smem>>>(d, nq, nc, eps, cyc, k, ld); cudaDeviceSynchronize(); }
  printf("NT %3d var %d ld %3d nq %3d nc %3d: k %3d  cycles %7lld  per step %6.0f  (%s)\n", NT, VAR, ld, nq, nc, *k, *cyc,
         (double)*cyc / (*k + 1), cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() {
  run<128, 0>(83, 15, 1e-9);  run<128, 1>(83, 15, 1e-9);
  run<512, 0>(83, 15, 1e-9);  run<512, 1>(83, 15, 1e-9);
  run<512, 0>(185, 31, 1e-9); run<512, 1>(185, 31, 1e-9);
  run<512, 0>(298, 60, 1e-9); run<512, 1>(298, 60, 1e-9);
  run<128, 0>(83, 15, 1e-9, true);
  run<512, 0>(185, 31, 1e-9, true); run<512, 0>(298, 60, 1e-9, true);
  return 0;
}
