// mcg_protocols.cuh — the reference's standalone protocol drivers on the
// device: Monte-Carlo pairing trials of the calcium-based
// bistable rule (gb_pairing_trial / gb_dp_curve, mechanisms.cpp:40-119) and
// the event-exact STDP window (stdp_window, mechanisms.cpp:9-38).
//
// Trials are independent, so each is one thread; everything data-dependent on
// the host side of the reference (the calcium jump schedule, sorted with
// std::sort; the pairing events, std::stable_sort) is built by the host code
// of this library with the same standard library calls on the same inputs,
// so the device replays exactly the reference's sequence.  Arithmetic follows
// the reference's expressions operation by operation (no contraction, the
// glibc-faithful exp and the reference's Threefry/Box-Muller draws).
#pragma once
#include "mcg_device.cuh"

struct McgGbDev {
  double tau_w, w_star, gamma_p, gamma_d, theta_p, theta_d, sigma;
  double r_tau_w;     // mcg_recip(tau_w)
  double cdecay;      // exp(-dt / tau_c)                         (mechanisms.cpp:70)
  double nz1, nz2;    // sigma * sqrt(k / tau_w) * sqrt(dt), k = 1, 2  (:81-82)
  double dt;
  uint64_t seed;
  int32_t trials, n_deltas;
};

// one thread per (delta index, trial)
__global__ void k_gb_trials(McgGbDev P, const int64_t* jstep, const double* jamt,
                            const int32_t* joff, const int64_t* nsteps, double* w0, double* wf) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= int64_t(P.trials) * P.n_deltas) return;
  const int di = int(i / P.trials), tr = int(i - int64_t(di) * P.trials);
  const mcg_key init_key = mcg_make_key(P.seed, uint64_t(tr), uint64_t(di), 0);
  const mcg_key noise_key = mcg_make_key(P.seed, uint64_t(tr), uint64_t(di), 1);
  double w = mcg_uniform_for(&init_key, 0) < 0.5 ? 0.0 : 1.0;
  w0[i] = w;
  double c = 0.0;
  int32_t jp = joff[di];
  const int32_t je = joff[di + 1];
  const int64_t n = nsteps[di];
  for (int64_t step = 0; step < n; ++step) {
    while (jp < je && jstep[jp] <= step) {
      c += jamt[jp];
      ++jp;
    }
    const bool hi = c > P.theta_p, lo = c > P.theta_d;
    // gb_drift (mechanisms.hpp:107-112)
    double d = -w * (1.0 - w) * (P.w_star - w);
    if (hi) d += P.gamma_p * (1.0 - w);
    if (lo) d -= P.gamma_d * w;
    double dw = mcg_div(d, P.tau_w, P.r_tau_w) * P.dt;
    if ((hi || lo) && P.sigma != 0.0) {
      const double nrm = mcg_normal_for(&noise_key, static_cast<uint64_t>(step));
      dw += ((hi && lo) ? P.nz2 : P.nz1) * nrm;
    }
    w += dw;
    c *= P.cdecay;
  }
  wf[i] = w;
}

struct McgStdpDev {
  double tau_pre, tau_post, a_pre, a_post, w0;
  int32_t n_deltas, n_pairs;
};

// one thread per delta: the sorted pairing events (t, pre) of that delta
__global__ void k_stdp_window(McgStdpDev P, const double* ev_t, const uint8_t* ev_pre,
                              const int32_t* ev_off, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n_deltas) return;
  double a_pre = 0.0, a_post = 0.0, w = P.w0, t_last = 0.0;
  for (int32_t e = ev_off[i]; e < ev_off[i + 1]; ++e) {
    const double dtm = ev_t[e] - t_last;  // stdp_decay (mechanisms.hpp:35-38)
    a_pre *= mcg_exp(-dtm / P.tau_pre);
    a_post *= mcg_exp(-dtm / P.tau_post);
    t_last = ev_t[e];
    if (ev_pre[e]) {  // stdp_on_pre / stdp_on_post (:40-48)
      a_pre += P.a_pre;
      w += a_post;
    } else {
      a_post += P.a_post;
      w += a_pre;
    }
  }
  out[i] = (w - P.w0) / P.n_pairs;
}
