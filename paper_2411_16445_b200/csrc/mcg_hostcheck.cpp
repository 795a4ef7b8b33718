// mcg_hostcheck.cpp — runtime check that this host's glibc libm is the one the
// device ports (mcg_libm.h + glibc_tables.h) were written against.
//
// Bitwise parity with the reference holds only when the reference's libm calls
// (exp: engine.cpp:44-54, :582, :601, :619, :671, :705-707; log/sincos:
// rng.cpp:62-64) run the same algorithm as the device ports: glibc 2.39's FMA
// ifunc variants (__exp_fma, __log_fma, __sincos_fma), tables extracted from
// the libm.so.6 with build-id kGlibcBuildId (gen_glibc_tables.py).  A host with
// another glibc build, or a CPU whose ifunc resolver picks the SSE2 variants,
// would run a reference that silently stops matching this engine.
//
// mcg_libm_check reports three facts: the build-id of the libm mapped into this
// process, whether the CPU has FMA + AVX2 (the resolver's condition for the FMA
// variants), and a differential run of the host build of the ports against the
// live libm on fixed pseudo-random arguments.  Built with -ffp-contract=off so
// the ports' host arithmetic is exactly their device arithmetic.
#include <dlfcn.h>
#include <link.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/mcg.h"
#include "mcg_libm.h"

namespace {

constexpr const char* kGlibcBuildId = "0d9969fe206760d250ec30a5a9be18aefbf84ea8";

struct BuildIdSearch {
  std::string path;
  std::string id;
};

int find_libm(struct dl_phdr_info* info, size_t, void* data) {
  auto* s = static_cast<BuildIdSearch*>(data);
  if (!info->dlpi_name || !std::strstr(info->dlpi_name, "libm.so")) return 0;
  s->path = info->dlpi_name;
  for (int i = 0; i < info->dlpi_phnum; ++i) {
    const ElfW(Phdr)& ph = info->dlpi_phdr[i];
    if (ph.p_type != PT_NOTE) continue;
    const auto* p = reinterpret_cast<const uint8_t*>(info->dlpi_addr + ph.p_vaddr);
    const uint8_t* end = p + ph.p_memsz;
    while (p + 12 <= end) {
      uint32_t namesz, descsz, type;
      std::memcpy(&namesz, p, 4);
      std::memcpy(&descsz, p + 4, 4);
      std::memcpy(&type, p + 8, 4);
      const uint8_t* name = p + 12;
      const uint8_t* desc = name + ((namesz + 3) & ~3u);
      if (type == 3 && namesz == 4 && std::memcmp(name, "GNU", 4) == 0) {
        char hex[3];
        for (uint32_t k = 0; k < descsz; ++k) {
          std::snprintf(hex, sizeof hex, "%02x", desc[k]);
          s->id += hex;
        }
        return 1;
      }
      p = desc + ((descsz + 3) & ~3u);
    }
  }
  return 1;
}

uint64_t g_sm;
uint64_t next64() {  // splitmix64
  uint64_t z = (g_sm += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
double unif(double lo, double hi) { return lo + (hi - lo) * (double(next64() >> 11) * 0x1p-53); }
bool same(double a, double b) { return mcg_asu(a) == mcg_asu(b) || (std::isnan(a) && std::isnan(b)); }

}  // namespace

extern "C" mcg_status mcg_libm_check(int64_t samples, char* report, int64_t cap) {
  // the live libm, called through pointers resolved at run time (no builtins,
  // no constant folding): these are the ifunc-resolved symbols the reference binds
  using F1 = double (*)(double);
  using F2 = void (*)(double, double*, double*);
  void* h = dlopen("libm.so.6", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libm.so.6", RTLD_NOW);
  F1 live_exp = h ? reinterpret_cast<F1>(dlsym(h, "exp")) : nullptr;
  F1 live_log = h ? reinterpret_cast<F1>(dlsym(h, "log")) : nullptr;
  F2 live_sincos = h ? reinterpret_cast<F2>(dlsym(h, "sincos")) : nullptr;

  BuildIdSearch s;
  dl_iterate_phdr(find_libm, &s);
  __builtin_cpu_init();
  const bool fma = __builtin_cpu_supports("fma") && __builtin_cpu_supports("avx2");

  long bad = 0, n = 0;
  if (live_exp && live_log && live_sincos) {
    g_sm = 0x6d6367u;
    const long m = samples > 0 ? static_cast<long>(samples) : 20000;
    const double er[][2] = {{-20, 20}, {-1, 1}, {-1e-3, 1e-3}, {-745.2, -700}, {700, 709.8}};
    for (const auto& r : er)
      for (long i = 0; i < m; ++i, ++n) {
        const double x = unif(r[0], r[1]);
        bad += !same(mcg_exp(x), live_exp(x));
      }
    for (long i = 0; i < m; ++i, n += 2) {
      const double u1 = (double(next64() >> 11) + 1.0) * 0x1p-53;  // Box–Muller's u1
      bad += !same(mcg_log(u1), live_log(u1));
      const double x = std::ldexp(unif(0.5, 1.0), int(next64() % 2000) - 1000);
      bad += !same(mcg_log(x), live_log(x));
    }
    for (long i = 0; i < m; ++i, n += 2) {
      const double x = double(next64() >> 11) * 0x1p-53 * 6.283185307179586;  // 2 pi u2
      double a, b, c, d;
      mcg_sincos(x, &a, &b);
      live_sincos(x, &c, &d);
      bad += !same(a, c) + !same(b, d);
    }
  }
  const bool id_ok = s.id == kGlibcBuildId;
  const bool ok = id_ok && fma && bad == 0 && n > 0;
  if (report && cap > 0)
    std::snprintf(report, static_cast<size_t>(cap),
                  "libm %s build-id %s (%s); cpu fma+avx2 %s; ports vs live libm: %ld/%ld differ",
                  s.path.empty() ? "?" : s.path.c_str(), s.id.empty() ? "?" : s.id.c_str(),
                  id_ok ? "matches the tables" : "DIFFERS from the tables' " "0d9969fe…",
                  fma ? "yes" : "NO (ifunc would pick the SSE2 variants)", bad, n);
  return ok ? MCG_OK : MCG_ERR_ENGINE;
}
