// eig.cu -- on-device FP64 Hermitian eigensolve of the F x F Casorati Gram.
//
// Replaces the small end of Eigen's JacobiSVD (svd.cpp:44): the right
// singular vectors of X are the eigenvectors of G = X^H X and sigma_j =
// sqrt(lambda_j).  Parallel cyclic Jacobi in one CTA: each round pairs all
// indices (round-robin tournament), computes the F/2 rotations
// J = diag(1, e^{-i phi}) R(c, s) from the current 2x2 diagonal blocks, then
// applies A <- J^H A J as independent 2x2 block updates and V <- V J.  The
// rotation formulas are those of oracle/fqf_oracle.c:oracle_heev.  Sweeps run
// until no pair exceeds the threshold |a_pq| <= 1e-16 sqrt(|a_pp a_qq|).
// A lives in shared memory when F^2 * 16 B fits, else in global memory (L2).
#include "common.cuh"

namespace fqfg {

constexpr int kEigThreads = 1024;
constexpr int kEigMaxF = 1024;

struct Rot {
  double c, s, er, ei;  // e = e^{-i phi}
};

__global__ void __launch_bounds__(kEigThreads) eig_kernel(double2* __restrict__ Ag, int F,
                                                          double* __restrict__ w_out,
                                                          double2* __restrict__ v_out,
                                                          double2* __restrict__ v_work,
                                                          int a_in_smem) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int m = F + (F & 1);  // even count with a dummy index F when F is odd
  const int h = m / 2;
  int* top = reinterpret_cast<int*>(smem_raw);
  int* bot = top + kEigMaxF / 2;
  Rot* rot = reinterpret_cast<Rot*>(bot + kEigMaxF / 2);
  int* flag = reinterpret_cast<int*>(rot + kEigMaxF / 2);
  double2* A = a_in_smem ? reinterpret_cast<double2*>(flag + 4) : Ag;  // flag[2..3]: fro
  double2* V = v_work;
  const int tid = threadIdx.x;

  if (a_in_smem)
    for (int i = tid; i < F * F; i += blockDim.x) A[i] = Ag[i];
  for (int i = tid; i < F * F; i += blockDim.x)
    V[i] = make_double2((i / F) == (i % F) ? 1.0 : 0.0, 0.0);
  for (int k = tid; k < h; k += blockDim.x) {
    top[k] = 2 * k;
    bot[k] = 2 * k + 1;
  }
  // Absolute floor for the rotation test: entries below 1e-20 ||A||_F carry no
  // information at the f32 precision the projection uses.
  double* fro = reinterpret_cast<double*>(flag + 2);
  if (tid == 0) *fro = 0.0;
  __syncthreads();
  {
    double s = 0.0;
    for (int i = tid; i < F * F; i += blockDim.x) {
      double2 v = A[i];
      s += v.x * v.x + v.y * v.y;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((tid & 31) == 0) atomicAdd(fro, s);
  }
  __syncthreads();
  const double tol_abs = 1e-20 * sqrt(*fro);

  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) flag[0] = 0;
    __syncthreads();
    for (int round = 0; round < m - 1; ++round) {
      for (int k = tid; k < h; k += blockDim.x) {
        int p = top[k], q = bot[k];
        if (p > q) {
          int t = p;
          p = q;
          q = t;
        }
        Rot r = {1.0, 0.0, 1.0, 0.0};
        if (q < F) {
          double2 apq = A[(size_t)p * F + q];
          double gm = hypot(apq.x, apq.y);
          double app = A[(size_t)p * F + p].x, aqq = A[(size_t)q * F + q].x;
          if (gm > tol_abs && gm > 1e-16 * sqrt(fabs(app * aqq))) {
            double zeta = (aqq - app) / (2.0 * gm);
            double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            r.c = 1.0 / sqrt(1.0 + t * t);
            r.s = r.c * t;
            r.er = apq.x / gm;
            r.ei = -apq.y / gm;
            flag[0] = 1;
          }
        }
        rot[k] = r;
      }
      __syncthreads();
      // A <- J^H A J over all 2x2 blocks (pair k rows, pair l cols).
      for (int b = tid; b < h * h; b += blockDim.x) {
        int k = b / h, l = b % h;
        int p = top[k], q = bot[k], pc = top[l], qc = bot[l];
        if (p > q) {
          int t = p;
          p = q;
          q = t;
        }
        if (pc > qc) {
          int t = pc;
          pc = qc;
          qc = t;
        }
        const Rot rk = rot[k], rl = rot[l];
        bool rq = q < F, cq = qc < F;
        double2 b00 = A[(size_t)p * F + pc];
        double2 b01 = cq ? A[(size_t)p * F + qc] : make_double2(0, 0);
        double2 b10 = rq ? A[(size_t)q * F + pc] : make_double2(0, 0);
        double2 b11 = (rq && cq) ? A[(size_t)q * F + qc] : make_double2(0, 0);
        // right: (x, y) -> (c x - s e y, s x + c e y)
        double2 t0, t1;
#define RIGHT(X_, Y_, o0, o1)                                          \
  {                                                                   \
    double eyr = rl.er * Y_.x - rl.ei * Y_.y;                         \
    double eyi = rl.er * Y_.y + rl.ei * Y_.x;                         \
    o0 = make_double2(rl.c * X_.x - rl.s * eyr, rl.c * X_.y - rl.s * eyi); \
    o1 = make_double2(rl.s * X_.x + rl.c * eyr, rl.s * X_.y + rl.c * eyi); \
  }
        RIGHT(b00, b01, t0, t1);
        b00 = t0;
        b01 = t1;
        RIGHT(b10, b11, t0, t1);
        b10 = t0;
        b11 = t1;
#undef RIGHT
        // left: (x; y) -> (c x - s conj(e) y ; s x + c conj(e) y)
#define LEFT(X_, Y_, o0, o1)                                           \
  {                                                                   \
    double eyr = rk.er * Y_.x + rk.ei * Y_.y;                         \
    double eyi = rk.er * Y_.y - rk.ei * Y_.x;                         \
    o0 = make_double2(rk.c * X_.x - rk.s * eyr, rk.c * X_.y - rk.s * eyi); \
    o1 = make_double2(rk.s * X_.x + rk.c * eyr, rk.s * X_.y + rk.c * eyi); \
  }
        LEFT(b00, b10, t0, t1);
        b00 = t0;
        b10 = t1;
        LEFT(b01, b11, t0, t1);
        b01 = t0;
        b11 = t1;
#undef LEFT
        if (k == l) {  // the pair's own block: exactly diagonal afterwards
          b01 = b10 = make_double2(0, 0);
          b00.y = b11.y = 0.0;
        }
        A[(size_t)p * F + pc] = b00;
        if (cq) A[(size_t)p * F + qc] = b01;
        if (rq) A[(size_t)q * F + pc] = b10;
        if (rq && cq) A[(size_t)q * F + qc] = b11;
      }
      // V <- V J (rows r, pair l).
      for (int b = tid; b < F * h; b += blockDim.x) {
        int r = b / h, l = b % h;
        int pc = top[l], qc = bot[l];
        if (pc > qc) {
          int t = pc;
          pc = qc;
          qc = t;
        }
        if (qc >= F) continue;
        const Rot rl = rot[l];
        double2 x = V[(size_t)r * F + pc], y = V[(size_t)r * F + qc];
        double eyr = rl.er * y.x - rl.ei * y.y, eyi = rl.er * y.y + rl.ei * y.x;
        V[(size_t)r * F + pc] = make_double2(rl.c * x.x - rl.s * eyr, rl.c * x.y - rl.s * eyi);
        V[(size_t)r * F + qc] = make_double2(rl.s * x.x + rl.c * eyr, rl.s * x.y + rl.c * eyi);
      }
      __syncthreads();
      // Round-robin: top[0] fixed; others rotate through top/bot.
      if (tid == 0) {
        int last_top = top[h - 1];
        for (int k = h - 1; k > 1; --k) top[k] = top[k - 1];
        if (h > 1) top[1] = bot[0];
        for (int k = 0; k < h - 1; ++k) bot[k] = bot[k + 1];
        if (h > 1) bot[h - 1] = last_top;
      }
      __syncthreads();
    }
    if (!flag[0]) break;
    __syncthreads();
  }

  // Sort eigenvalues descending (stable rank), permute eigenvector columns.
  for (int i = tid; i < F; i += blockDim.x) {
    double wi = A[(size_t)i * F + i].x;
    int rank = 0;
    for (int j = 0; j < F; ++j) {
      double wj = A[(size_t)j * F + j].x;
      rank += (wj > wi) || (wj == wi && j < i);
    }
    w_out[rank] = wi;
    for (int r = 0; r < F; ++r) v_out[(size_t)r * F + rank] = V[(size_t)r * F + i];
  }
}

}  // namespace fqfg
