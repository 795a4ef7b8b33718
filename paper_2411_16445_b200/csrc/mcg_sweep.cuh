// mcg_sweep.cuh — the constant-diagonal Hines solve (V, or one species, of one
// cell) scheduled along the tree's chains, one lane per chain.
//
// tree_solver.cpp:46-74 eliminates leaves-to-root in descending index order,
// rhs[par[i]] += f[i]*rhs[i], then substitutes root-to-leaves,
// v[i] = (rhs[i] + coupling[i]*v[par[i]]) / diag[i].  With the diagonal
// constant (McgKind::v_const / sp_const) f and the eliminated diagonal d are
// precomputed, and what is left per step are two dependent chains of fp64
// operations through the tree.  For a "spider" tree — every node but the root
// has at most one child, the shape of the consolidation cells (soma halves
// continued by an apical and a basal dendrite) — each chain
// hanging off the root depends only on itself, so the two chains of a system
// run on two adjacent lanes and meet at the root through one shuffle: the
// latency is the longer chain, not the node count.
//
// Every fp64 operation is the reference's, with the reference's operands:
//   r2[i]  = cap[i]*x[i] + rhs[i]                   (tree_solver.cpp:57)
//   r2[p] += f[c]*r2[c]   for the only child c of p  (:66): along a chain the
//            running value is final once its predecessor is; the root adds its
//            children's terms in descending child order, as the loop does
//   x[i]   = (r2[i] + coup[i]*x[par[i]]) / d[i]     (:71-73)
// The chains are stored position-major, leaf side padded to a multiple of 4
// and tops aligned (mcg_build.cpp chain_schedule); padding positions carry
// f = -0, coup = 0, d = y = 1 and r2 = +0, which are exact identities
// ((-0)*x + r == r and +0 + (+-0) == +0 in round-to-nearest).
// The division is Markstein's correctly rounded quotient from y = RN(1/d)
// (mcg_div, mcg_device.cuh) without the per-division range test on the
// dependent chain: the numerators' range is checked off the chain and if any
// lies outside [2^-700, 2^700] (other than +0) the pair redoes its
// substitution with IEEE division from the stored r2.  The host guarantees
// d in [2^-200, 2^200] for these systems (McgKind::ch_lp > 0).
#pragma once
#include <stdint.h>

extern __shared__ double mcg_smem[];

// numerator outside the range where the reciprocal quotient is exact (or -0)
__device__ __forceinline__ unsigned mcg_div_bad(double num) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(num));
  const unsigned long long a = b & 0x7fffffffffffffffull;
  constexpr unsigned long long lo = 0x1430000000000000ull;  // 2^-700
  constexpr unsigned long long hi = 0x6bb0000000000000ull;  // 2^700
  return (b != 0ull && a - lo > hi - lo) ? 1u : 0u;
}

__device__ __forceinline__ double mcg_qdiv(double x, double d, double y) {
  const double q = __dmul_rn(x, y);
  const double r = __fma_rn(-q, d, x);
  return __fma_rn(r, y, q);
}

// one lane of the chain sweep (offsets into mcg_smem; idx in int32 units)
struct McgChainLane {
  int on;        // this lane's system takes the chain sweep this step
  int side;      // 0: chain A (positions [0, lp)), 1: chain B ([lp, 2 lp))
  int lp;        // positions per chain (multiple of 4); the root is at 2 lp
  int r2c;       // r2 after elimination, by position
  int fc;        // f | coup | d | y | cap | g_leak_rhs, by position, each 2 lp + 1 long
  int idx;       // position -> node (-1: padding)
  int x;         // solved state, by node
  int a_first;   // chain A's top has the larger index
  int v;         // V system (else species)
  int rc;        // V: rhs_current by node (-1: no current this step)
  int pc;        // species: synthesis compartment (-1: no production)
  double prod;   // species: production at pc
};

// r2 of a position before elimination, cap*x + rhs (tree_solver.cpp:57), with
// the reference's right-hand sides (engine.cpp:683 / 746-748); padding
// positions (node < 0) give +0
__device__ __forceinline__ double mcg_chain_rinit(const McgChainLane& L, int node, double cap,
                                                  double gl, double x, double rc) {
  const double rhs = L.v ? (gl + 0.0 + (L.rc >= 0 ? rc : 0.0)) : (node == L.pc ? L.prod : 0.0);
  return cap * x + rhs;
}

// all 32 lanes of the warp must call this (inactive lanes with on = 0)
__device__ __forceinline__ void mcg_chain_lane(const McgChainLane& L) {
  double* S = mcg_smem;
  const int32_t* PI = reinterpret_cast<const int32_t*>(mcg_smem);
  const int lp = L.on ? L.lp : 0;
  const int P = 2 * L.lp + 1;
  const int p0 = L.side * L.lp;
  const int rb = L.r2c + p0, fb = L.fc + p0, cb = L.fc + P + p0, db = L.fc + 2 * P + p0,
            yb = L.fc + 3 * P + p0, ib = L.idx + p0;

  // ---- elimination, leaf side first.  Block b's links run while block b + 4's
  // r2 is formed from operands loaded one block ahead, whose node indices were
  // loaded two blocks ahead
  const int capb = L.fc + 4 * P + p0, glb = L.fc + 5 * P + p0;
  double cur = 0.0, fp = -0.0;
  {
    double r4[4], f4[4];
    int i4[4];  // node indices of the block after the one r4 holds
    auto load_idx = [&](int b, int* o) {
#pragma unroll
      for (int u = 0; u < 4; ++u) o[u] = (b < lp) ? PI[ib + b + u] : -1;
    };
    auto form = [&](int b, const int* id, double* r, double* f) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int node = id[u];
        const double x = node >= 0 ? S[L.x + node] : 0.0;
        const double rc = (node >= 0 && L.rc >= 0) ? S[L.rc + node] : 0.0;
        const double gl = L.v ? S[glb + b + u] : 0.0;
        r[u] = mcg_chain_rinit(L, node, S[capb + b + u], gl, x, rc);
        f[u] = S[fb + b + u];
      }
    };
    if (lp > 0) {
      int i0[4];
      load_idx(0, i0);
      load_idx(4, i4);
      form(0, i0, r4, f4);
    }
#pragma unroll 1
    for (int b = 0; b < lp; b += 4) {
      int in[4];
      load_idx(b + 8, in);
      double rn[4], fn[4];
      const int nb = (b + 4 < lp) ? b + 4 : b;  // the last block forms itself again (unused)
      form(nb, i4, rn, fn);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double r = r4[u] + fp * cur;
        S[rb + b + u] = r;
        cur = r;
        fp = f4[u];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        r4[u] = rn[u];
        f4[u] = fn[u];
        i4[u] = in[u];
      }
    }
  }
  // ---- root: the children's terms in descending child order
  const double t = fp * cur;  // f of this chain's top times its final r2
  const double to = __shfl_xor_sync(0xffffffffu, t, 1);
  const double ta = L.side == 0 ? t : to, tb = L.side == 0 ? to : t;
  double r0 = 0.0;
  if (L.on) {
    const int pr = L.fc + 2 * L.lp;  // root position
    r0 = mcg_chain_rinit(L, 0, S[pr + 4 * P], L.v ? S[pr + 5 * P] : 0.0, S[L.x],
                         L.rc >= 0 ? S[L.rc] : 0.0);
  }
  if (L.a_first) {
    r0 = r0 + ta;
    r0 = r0 + tb;
  } else {
    r0 = r0 + tb;
    r0 = r0 + ta;
  }
  // ---- substitution, top first
  unsigned bad = L.on ? mcg_div_bad(r0) : 0u;
  double xv = 0.0;
  if (L.on) {
    xv = mcg_qdiv(r0, S[L.fc + 2 * P + 2 * L.lp], S[L.fc + 3 * P + 2 * L.lp]);
    if (L.side == 0) S[L.x] = xv;
  }
  {
    // blocks of two positions (register budget), next block loaded ahead
    double r2v[2], c2v[2], d2v[2], y2v[2];
    int i2v[2];
    if (lp > 0) {
      const int b = lp - 2;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        r2v[u] = S[rb + b + u];
        c2v[u] = S[cb + b + u];
        d2v[u] = S[db + b + u];
        y2v[u] = S[yb + b + u];
        i2v[u] = PI[ib + b + u];
      }
    }
#pragma unroll 1
    for (int b = lp - 2; b >= 0; b -= 2) {
      double rn[2], cn[2], dn[2], yn[2];
      int in[2];
      const int nb = b >= 2 ? b - 2 : b;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        rn[u] = S[rb + nb + u];
        cn[u] = S[cb + nb + u];
        dn[u] = S[db + nb + u];
        yn[u] = S[yb + nb + u];
        in[u] = PI[ib + nb + u];
      }
#pragma unroll
      for (int u = 1; u >= 0; --u) {
        const double num = r2v[u] + c2v[u] * xv;
        bad |= mcg_div_bad(num);
        xv = mcg_qdiv(num, d2v[u], y2v[u]);
        if (i2v[u] >= 0) S[L.x + i2v[u]] = xv;
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        r2v[u] = rn[u];
        c2v[u] = cn[u];
        d2v[u] = dn[u];
        y2v[u] = yn[u];
        i2v[u] = in[u];
      }
    }
  }
  bad |= __shfl_xor_sync(0xffffffffu, bad, 1);
  if (bad && L.on) {  // rare: the substitution again with IEEE division
    double xe = __ddiv_rn(r0, S[L.fc + 2 * P + 2 * L.lp]);
    if (L.side == 0) S[L.x] = xe;
    for (int p = lp - 1; p >= 0; --p) {
      xe = __ddiv_rn(S[rb + p] + S[cb + p] * xe, S[db + p]);
      const int i = PI[ib + p];
      if (i >= 0) S[L.x + i] = xe;
    }
  }
}
