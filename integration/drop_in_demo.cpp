// drop_in_demo.cpp — the reference's own recipe builders through both
// mcsim::Engine (the unmodified reference, oracle/_ref) and the drop-in
// mcsim_gpu::Engine (integration/mcsim_gpu.hpp over libmcg.so); exits 0 iff
// spike trains and sampled cell state are bitwise identical.
//   drop_in_demo [consolidation|busyring] [t_ms]
// Test infrastructure (tests/test_gpu_dropin.py); built by _build.py when the
// reference headers are present.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "mcsim/bench.hpp"
#include "mcsim/network.hpp"
#include "mcsim_gpu.hpp"

// spikes and sampled cell state of both engines after advance_to(t_ms)
template <class A, class B>
static int compare_state(A& ref, B& gpu, const mcsim::Recipe& r, double t_ms) {
  ref.advance_to(t_ms);
  gpu.advance_to(t_ms);
  const auto& s0 = ref.spikes();
  const auto& s1 = gpu.spikes();
  if (s0.size() != s1.size()) {
    std::printf("FAIL spike count %zu vs %zu\n", s0.size(), s1.size());
    return 1;
  }
  for (std::size_t i = 0; i < s0.size(); ++i)
    if (s0[i].gid != s1[i].gid || std::memcmp(&s0[i].t_ms, &s1[i].t_ms, 8) != 0) {
      std::printf("FAIL spike %zu: (%u, %.17g) vs (%u, %.17g)\n", i, s0[i].gid, s0[i].t_ms,
                  s1[i].gid, s1[i].t_ms);
      return 1;
    }
  const uint32_t n = static_cast<uint32_t>(r.cell_kind.size());
  for (uint32_t gid = 0; gid < n; gid += (n > 16 ? n / 16 : 1)) {
    const auto& a = ref.cell(gid);
    const auto& b = gpu.cell(gid);
    if (a.v_mV != b.v_mV || a.species != b.species) {
      std::printf("FAIL cell %u membrane/species state\n", gid);
      return 1;
    }
    for (std::size_t g = 0; g < a.groups.size(); ++g)
      for (std::size_t i = 0; i < a.groups[g].stc.size(); ++i) {
        const auto &x = a.groups[g].stc[i], &y = b.groups[g].stc[i];
        if (std::memcmp(&x, &y, sizeof x) != 0) {
          std::printf("FAIL cell %u group %zu STC instance %zu\n", gid, g, i);
          return 1;
        }
      }
  }
  return 0;
}

template <class A, class B>
static int compare(A& ref, B& gpu, const mcsim::Recipe& r, double t_ms) {
  if (const int rc = compare_state(ref, gpu, r, t_ms)) return rc;
  const std::size_t n_spikes = ref.spikes().size();
  const uint32_t n = static_cast<uint32_t>(r.cell_kind.size());
  // checkpoints: the same MCSCKPT1 bytes, and each engine restores the other's
  const auto b0 = ref.make_checkpoint().serialize();
  const auto b1 = gpu.make_checkpoint().serialize();
  if (b0 != b1) {
    std::printf("FAIL checkpoints differ (%zu vs %zu bytes)\n", b0.size(), b1.size());
    return 1;
  }
  // restore over a diverged state that has a live cell() mirror: the mirror
  // must be dropped, not written back over the restored state
  gpu.advance_to(t_ms + 100.0);
  (void)gpu.cell(0);
  gpu.restore(mcsim::Checkpoint::deserialize(b0));
  if (gpu.cell(0).v_mV != ref.cell(0).v_mV) {
    std::printf("FAIL cell 0 after restore returns the pre-restore mirror\n");
    return 1;
  }
  ref.clear_spikes();
  gpu.clear_spikes();
  const double t2 = t_ms + 200.0;
  ref.advance_to(t2);
  gpu.advance_to(t2);
  const auto& r0 = ref.spikes();
  const auto& r1 = gpu.spikes();
  bool same = r0.size() == r1.size();
  for (std::size_t i = 0; same && i < r0.size(); ++i)
    same = r0[i].gid == r1[i].gid && std::memcmp(&r0[i].t_ms, &r1[i].t_ms, 8) == 0;
  for (uint32_t gid = 0; same && gid < n; gid += (n > 16 ? n / 16 : 1))
    same = ref.cell(gid).v_mV == gpu.cell(gid).v_mV && ref.cell(gid).species == gpu.cell(gid).species;
  if (!same) {
    std::printf("FAIL continuation after restore differs (%zu vs %zu spikes)\n", r0.size(), r1.size());
    return 1;
  }
  std::printf("OK %zu spikes identical, checkpoints identical (%zu bytes), t = %.1f ms; "
              "restore + %zu spikes to %.1f ms identical\n",
              n_spikes, b0.size(), t_ms, r0.size(), t2);
  return 0;
}

// a malformed recipe through both engines: the same exception type and text
template <class E>
static std::string build_error(const mcsim::Recipe& r, const mcsim::EngineOptions& opt) {
  try {
    E e(r, opt);
  } catch (const mcsim::EngineError& x) {
    return std::string("EngineError: ") + x.what();
  } catch (const std::exception& x) {
    return std::string("other: ") + x.what();
  }
  return "no error";
}

static int errors() {
  mcsim::ConsolidationConfig cfg;
  cfg.n_cells = 20;
  cfg.n_exc = 16;
  cfg.pattern = 4;
  mcsim::ConsolidationBuild b = mcsim::build_consolidation_network(cfg, false);
  const mcsim::EngineOptions opt{cfg.dt_ms, cfg.seed, 1};
  b.recipe.connections.at(3).label = "no_such_label";
  const std::string e0 = build_error<mcsim::Engine>(b.recipe, opt);
  const std::string e1 = build_error<mcsim_gpu::Engine>(b.recipe, opt);
  if (e0 != e1 || e0.find("no_such_label") == std::string::npos) {
    std::printf("FAIL build errors differ: '%s' vs '%s'\n", e0.c_str(), e1.c_str());
    return 1;
  }
  std::printf("OK both engines: %s\n", e0.c_str());
  return 0;
}

int main(int argc, char** argv) {
  const std::string which = argc > 1 ? argv[1] : "consolidation";
  const double t_ms = argc > 2 ? std::atof(argv[2]) : 2000.0;
  try {
    if (which == "errors") return errors();
    if (which == "busyring") {
      mcsim::BusyringSpec spec = mcsim::default_busyring();
      spec.n_cells = 256;
      spec.ring_weight_uS = mcsim::calibrate_ring_weight(spec);
      const mcsim::Recipe r = mcsim::build_busyring(spec);
      const mcsim::EngineOptions opt{spec.dt_ms, spec.seed, 8};
      mcsim::Engine ref(r, opt);
      mcsim_gpu::Engine gpu(r, opt);
      return compare(ref, gpu, r, t_ms);
    }
    mcsim::ConsolidationConfig cfg;
    cfg.seed = 1;
    cfg.multi_compartment = true;
    const mcsim::ConsolidationBuild b = mcsim::build_consolidation_network(cfg, true);
    const mcsim::EngineOptions opt{cfg.dt_ms, cfg.seed, 8};
    mcsim::Engine ref(b.recipe, opt);
    if (which == "sharded") {
      // the shard constructor with a one-rank communicator: the exchange runs
      // inside libmcg (stepping launch + ncclAllGather per epoch)
      mcsim_gpu::Shard sh;
      sh.nccl_id = mcsim_gpu::nccl_unique_id();
      mcsim_gpu::Engine gpu(b.recipe, opt, sh);
      const int rc = compare_state(ref, gpu, b.recipe, t_ms);
      if (rc == 0) std::printf("OK sharded: %zu spikes identical, t = %.1f ms\n", gpu.spikes().size(), t_ms);
      return rc;
    }
    mcsim_gpu::Engine gpu(b.recipe, opt);
    return compare(ref, gpu, b.recipe, t_ms);
  } catch (const std::exception& e) {
    std::printf("ERROR %s\n", e.what());
    return 2;
  }
}
