// mcg_mech.cuh — per-cell mechanism helpers shared by the epoch and
// fast-forward kernels: active-list kernel decay with the reference's ordered
// conductance/current folds (engine.cpp:578-616), the post-spike hook
// (engine.cpp:515-539), and the fast-forward entry checks (engine.cpp:958-969).
#pragma once
#include "mcg_device.cuh"


// decay an active list, fold kept kernels in active-list order (engine.cpp:578-616).
// Every instance of a group sits on the placement's compartment `comp`
// (append_instance(g, pl.comp, ...), engine.cpp:330-372), so the fold is one
// running sum (two for conductances) in registers, read and written once.  A
// chunk of 32 kernels is folded lane by lane from shuffles: dropped kernels
// contribute -0.0, the identity of fp64 addition, so dense chunks need no
// per-lane branch; sparse chunks (few kept) take only the kept lanes.
__device__ __forceinline__ bool mcg_decay_active(const McgDev& D, McgCellGroup* G, double f,
                                                 bool cond, double* acc, double* acc2,
                                                 double erev, int comp, int lane) {
  const int na = G->active_n;
  if (na == 0) return false;
  const int64_t base = G->inst;
  int out = 0;
  double r1 = acc[comp];
  double r2 = cond ? acc2[comp] : 0.0;
  // loads run ahead of the chunk being folded: kernels one chunk, indices two
  int i_cur = lane < na ? D.i_active[base + lane] : 0;
  double k_cur = lane < na ? D.i_kernel[base + i_cur] : 0.0;
  int i_nx = lane + 32 < na ? D.i_active[base + lane + 32] : 0;
  for (int a0 = 0; a0 < na; a0 += 32) {
    const int a = a0 + lane;
    const int i = i_cur;
    const double k_nx = (a + 32 < na) ? D.i_kernel[base + i_nx] : 0.0;
    const int i_nx2 = (a + 64 < na) ? D.i_active[base + a + 64] : 0;
    double kv = 0.0;
    bool keep = false;
    if (a < na) {
      kv = k_cur * f;
      if (cond ? (kv < 1e-30) : (fabs(kv) < 1e-30)) kv = 0.0;
      D.i_kernel[base + i] = kv;
      keep = kv != 0.0;
    }
    i_cur = i_nx;
    k_cur = k_nx;
    i_nx = i_nx2;
    const unsigned m = __ballot_sync(MCG_FULL, keep);
    // compaction: the slots written, [out, out + popc), lie below a0 + 32,
    // and the next two chunks' indices are already in registers
    if (keep) D.i_active[base + out + __popc(m & mcg_lanemask_lt())] = i;
    const double c1 = keep ? kv : -0.0;
    const double c2 = keep ? kv * erev : -0.0;
    if (__popc(m) > 8) {
#pragma unroll
      for (int l = 0; l < 32; ++l) {
        r1 += __shfl_sync(MCG_FULL, c1, l);
        if (cond) r2 += __shfl_sync(MCG_FULL, c2, l);
      }
    } else {
      for (unsigned mm = m; mm; mm &= mm - 1) {
        const int l = __ffs(mm) - 1;
        r1 += __shfl_sync(MCG_FULL, c1, l);
        if (cond) r2 += __shfl_sync(MCG_FULL, c2, l);
      }
    }
    out += __popc(m);
  }
  __syncwarp();
  if (lane == 0) {
    acc[comp] = r1;  // r1 + (-0.0) * k == r1: unchanged when nothing was kept
    if (cond) acc2[comp] = r2;
    G->active_n = out;
  }
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

