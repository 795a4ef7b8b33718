// mcg_mech.cuh — per-cell mechanism helpers shared by the epoch and
// fast-forward kernels: active-list kernel decay with the reference's ordered
// conductance/current folds (engine.cpp:578-616), the post-spike hook
// (engine.cpp:515-539), and the fast-forward entry checks (engine.cpp:958-969).
#pragma once
#include "mcg_device.cuh"


// decay an active list, fold kept kernels in active-list order (engine.cpp:578-616)
__device__ __forceinline__ bool mcg_decay_active(const McgDev& D, McgCellGroup* G, double f,
                                                 bool cond, double* acc, double* acc2,
                                                 double erev, int lane) {
  const int na = G->active_n;
  const int64_t base = G->inst;
  int out = 0;
  // the reference's in-order fold acc[comp] += kv (and acc2[comp] += kv * erev),
  // run by every lane on shuffled values with the running sums in registers
  // while consecutive kernels share a compartment (they usually all do)
  int rc = -1;
  double r1 = 0.0, r2 = 0.0;
  for (int a0 = 0; a0 < na; a0 += 32) {
    const int a = a0 + lane;
    int i = 0, comp = 0;
    double kv = 0.0;
    bool keep = false;
    if (a < na) {
      i = D.i_active[base + a];
      const int64_t j = base + i;
      kv = D.i_kernel[j] * f;
      if (cond ? (kv < 1e-30) : (fabs(kv) < 1e-30)) kv = 0.0;
      D.i_kernel[j] = kv;
      keep = kv != 0.0;
      comp = D.i_comp[j];
    }
    const unsigned m = __ballot_sync(MCG_FULL, keep);
    __syncwarp();
    if (keep) D.i_active[base + out + __popc(m & mcg_lanemask_lt())] = i;
    unsigned mm = m;
    while (mm) {
      // up to four kept kernels per batch of shuffles, folded in order
      int l[4];
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        l[u] = mm ? __ffs(mm) - 1 : 0;
        if (mm) {
          mm &= mm - 1;
          cnt = u + 1;
        }
      }
      double kl[4];
      int cl[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        kl[u] = __shfl_sync(MCG_FULL, kv, l[u]);
        cl[u] = __shfl_sync(MCG_FULL, comp, l[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (u >= cnt) break;
        if (cl[u] != rc) {
          if (rc >= 0 && lane == 0) {
            acc[rc] = r1;
            if (cond) acc2[rc] = r2;
          }
          __syncwarp();
          rc = cl[u];
          r1 = acc[rc];
          if (cond) r2 = acc2[rc];
        }
        r1 += kl[u];
        if (cond) r2 += kl[u] * erev;
      }
    }
    out += __popc(m);
  }
  if (rc >= 0 && lane == 0) {
    acc[rc] = r1;
    if (cond) acc2[rc] = r2;
  }
  __syncwarp();
  if (lane == 0) G->active_n = out;
  __syncwarp();
  return out > 0;
}

// post_event (engine.cpp:515-539): every synapse of the cell, lanes in parallel
__device__ __forceinline__ void mcg_post_event(const McgDev& D, const McgKind& K, int64_t cg0,
                                               int64_t s, int lane) {
  for (int gi = 0; gi < K.n_groups; ++gi) {
    const McgCellGroup G = D.cgs[cg0 + gi];
    const McgSpec& S = D.specs[G.spec];
    if (S.kind == MCG_SYN_STDP_COND) {
      for (int i = lane; i < G.size; i += 32) {
        const int64_t j = G.inst + i;
        double pre = D.i_stdp_pre[j], post = D.i_stdp_post[j];
        const double gap = double(s + 1 - D.i_stdp_last[j]) * D.dt;
        if (gap > 0) mcg_stdp_decay(pre, post, S, gap);
        D.i_stdp_last[j] = s + 1;
        post += S.a_post;  // stdp_on_post
        D.i_stdp_w[j] += pre;
        D.i_stdp_pre[j] = pre;
        D.i_stdp_post[j] = post;
      }
    } else if (S.kind == MCG_SYN_HOMEO_CURRENT) {
      for (int i = lane; i < G.size; i += 32) {
        const int64_t j = G.inst + i;
        D.i_homeo_w[j] = fmax(D.i_homeo_w[j] + S.dw_minus, 0.0);
      }
    } else if (S.kind == MCG_SYN_STC_CHARGE) {
      for (int i = lane; i < G.size; i += 32) D.i_stc_c[G.inst + i] += S.cpost_s;
    }
  }
}

// ---------------------------------------------------------------------------
// fast-forward (engine.cpp:947-1034)
// ---------------------------------------------------------------------------
__global__ void k_ff_pending(McgDev D, int32_t n_fifos, int32_t* flag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_fifos && D.fifos[i].head < D.fifos[i].tail) atomicOr(flag, 1);
}

// zero calcium, STDP traces, kernels and active lists (engine.cpp:961-969)
__global__ void k_ff_reset(McgDev D, int64_t n_cg) {
  const int64_t g = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g >= n_cg) return;
  McgCellGroup& G = D.cgs[g];
  const McgSpec& S = D.specs[G.spec];
  for (int i = 0; i < G.size; ++i) {
    const int64_t j = G.inst + i;
    if (S.kind == MCG_SYN_STC_CHARGE) D.i_stc_c[j] = 0.0;
    if (S.kind == MCG_SYN_STDP_COND) {
      D.i_stdp_pre[j] = 0.0;
      D.i_stdp_post[j] = 0.0;
    }
    D.i_kernel[j] = 0.0;
  }
  G.active_n = 0;
}

