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
  // register mode (mcg_chain_lane<false>): the only nonzero rhs_current of a
  // step is at node rc_node (-2: no current), value rc_val = 0.0 + I (the
  // zero-filled buffer plus the one current, engine.cpp:575/662)
  int rc_node;
  double rc_val;
};

// r2 of a position before elimination, cap*x + rhs (tree_solver.cpp:57), with
// the reference's right-hand sides (engine.cpp:683 / 746-748); padding
// positions (node < 0) give +0
__device__ __forceinline__ double mcg_chain_rinit(const McgChainLane& L, int node, double cap,
                                                  double gl, double x, double rc) {
  const double rhs = L.v ? (gl + 0.0 + (L.rc >= 0 ? rc : 0.0)) : (node == L.pc ? L.prod : 0.0);
  return cap * x + rhs;
}

// register mode: rc is the node's rhs_current (0.0 off the current's node);
// gl + 0.0 + 0.0 == gl + 0.0 for every gl, so the V right-hand side is the
// reference's whether or not the step has a current
__device__ __forceinline__ double mcg_chain_rinit_reg(const McgChainLane& L, int node, double cap,
                                                      double gl, double x, double rc) {
  const double rhs = L.v ? (gl + 0.0 + rc) : (node == L.pc ? L.prod : 0.0);
  return cap * x + rhs;
}

// all 32 lanes of the warp must call this (inactive lanes with on = 0).
// Two passes over the lane's chain side, so that the two dependent chains
// carry nothing but their own fp64 operations:
//   1+2. elimination, leaf to top: r2[p] += f[c]*r2[c] along the chain, with
//        r2 = cap*x + rhs of the next block formed (off the chain) while the
//        current block's links run
//   3.   the root, then substitution, top to leaf, with the reciprocal quotient
// Each chain loop loads the next block's operands before the current block's
// links, so the shared-memory latency stays off the chain.
template <bool kRcBuf = true>
__device__ __forceinline__ void mcg_chain_lane(const McgChainLane& L) {
  double* S = mcg_smem;
  const int32_t* PI = reinterpret_cast<const int32_t*>(mcg_smem);
  const int lp = L.on ? L.lp : 0;
  const int P = 2 * L.lp + 1;
  const int p0 = L.side * L.lp;
  const int rb = L.r2c + p0, fb = L.fc + p0, cb = L.fc + P + p0, db = L.fc + 2 * P + p0,
            yb = L.fc + 3 * P + p0, ib = L.idx + p0;
  const int capb = L.fc + 4 * P + p0, glb = L.fc + 5 * P + p0;
  // the root's state, read before the root shuffle: side 0 stores the root's
  // new value right after it, and the two lanes need not be converged there
  const double x_root = L.on ? S[L.x] : 0.0;
  const double rc_root = kRcBuf ? ((L.on && L.rc >= 0) ? S[L.rc] : 0.0) : (L.rc_node == 0 ? L.rc_val : 0.0);

  // ---- 1 + 2. r2 = cap*x + rhs (tree_solver.cpp:57; padding positions +0)
  // formed for the block ahead while the current block's links run, then the
  // elimination, leaf to top: r2[p] += f[c]*r2[c] along the chain.  cur = the
  // final r2 of the last position, fp its f (the child's factor applied to
  // its parent).  Two register blocks in turn.
  auto r2_block = [&](int b, double* r, double* f) {
    int nd[4];
    double xv[4], rcv[4], cp[4], gl[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      nd[u] = PI[ib + b + u];
      cp[u] = S[capb + b + u];
      gl[u] = S[glb + b + u];
      f[u] = S[fb + b + u];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = nd[u] >= 0 ? nd[u] : 0;  // padding reads node 0 and discards it
      xv[u] = S[L.x + q];
      rcv[u] = kRcBuf ? S[(L.rc >= 0 ? L.rc : L.x) + q] : (nd[u] == L.rc_node ? L.rc_val : 0.0);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double v = kRcBuf ? mcg_chain_rinit(L, nd[u], cp[u], gl[u], xv[u], rcv[u])
                              : mcg_chain_rinit_reg(L, nd[u], cp[u], gl[u], xv[u], rcv[u]);
      r[u] = nd[u] >= 0 ? v : 0.0;
    }
  };
  double cur = 0.0, fp = -0.0;
  if (lp > 0) {
    double rA[4], fA[4], rB[4], fB[4];
    r2_block(0, rA, fA);
#pragma unroll 1
    for (int b = 0; b < lp; b += 8) {
      const bool two = b + 4 < lp;
      const int nb = two ? b + 4 : b;
      r2_block(nb, rB, fB);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double r = rA[u] + fp * cur;
        S[rb + b + u] = r;
        cur = r;
        fp = fA[u];
      }
      if (!two) break;
      const int na = b + 8 < lp ? b + 8 : b;
      r2_block(na, rA, fA);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double r = rB[u] + fp * cur;
        S[rb + b + 4 + u] = r;
        cur = r;
        fp = fB[u];
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
    r0 = kRcBuf ? mcg_chain_rinit(L, 0, S[pr + 4 * P], L.v ? S[pr + 5 * P] : 0.0, x_root, rc_root)
                : mcg_chain_rinit_reg(L, 0, S[pr + 4 * P], L.v ? S[pr + 5 * P] : 0.0, x_root, rc_root);
  }
  if (L.a_first) {
    r0 = r0 + ta;
    r0 = r0 + tb;
  } else {
    r0 = r0 + tb;
    r0 = r0 + ta;
  }
  // ---- 3. substitution, top first
  unsigned bad = L.on ? mcg_div_bad(r0) : 0u;
  double xv = 0.0;
  if (L.on) {
    xv = mcg_qdiv(r0, S[L.fc + 2 * P + 2 * L.lp], S[L.fc + 3 * P + 2 * L.lp]);
    if (L.side == 0) S[L.x] = xv;
  }
  if (lp > 0) {
    // two register blocks in turn, as the elimination
    double rA[4], cA[4], dA[4], yA[4], rB[4], cB[4], dB[4], yB[4];
    int iA[4], iB[4];
    auto load = [&](int b, double* r, double* c, double* d, double* y, int* i) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        r[u] = S[rb + b + u];
        c[u] = S[cb + b + u];
        d[u] = S[db + b + u];
        y[u] = S[yb + b + u];
        i[u] = PI[ib + b + u];
      }
    };
    auto links = [&](const double* r, const double* c, const double* d, const double* y,
                     const int* i) {
#pragma unroll
      for (int u = 3; u >= 0; --u) {
        const double num = r[u] + c[u] * xv;
        bad |= mcg_div_bad(num);
        xv = mcg_qdiv(num, d[u], y[u]);
        if (i[u] >= 0) S[L.x + i[u]] = xv;
      }
    };
    load(lp - 4, rA, cA, dA, yA, iA);
#pragma unroll 1
    for (int b = lp - 4; b >= 0; b -= 8) {
      const bool two = b >= 4;
      load(two ? b - 4 : b, rB, cB, dB, yB, iB);
      links(rA, cA, dA, yA, iA);
      if (!two) break;
      load(b >= 8 ? b - 8 : b, rA, cA, dA, yA, iA);
      links(rB, cB, dB, yB, iB);
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
