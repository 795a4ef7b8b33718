// ref_csv.cpp — TEST INFRASTRUCTURE ONLY: the reference's own CSV writers
// (csvio.cpp:34-69, compiled from /root/reference/proj/src/csvio.cpp by
// oracle/build_ref.sh) on arrays read from a binary file:
//   ref_csv spikes|trace <in.bin> <out.csv>
// in.bin = int64 n, n doubles (t_s), then n uint32 gids (spikes) or n doubles.
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#include "mcsim/csvio.hpp"

int main(int argc, char** argv) {
  if (argc != 4) return 2;
  FILE* f = std::fopen(argv[2], "rb");
  if (!f) return 3;
  int64_t n = 0;
  if (std::fread(&n, 8, 1, f) != 1) return 4;
  std::vector<double> t(n);
  if (n && std::fread(t.data(), 8, n, f) != size_t(n)) return 5;
  if (std::strcmp(argv[1], "spikes") == 0) {
    mcsim::SpikeData d;
    d.t_s = t;
    d.gid.resize(n);
    if (n && std::fread(d.gid.data(), 4, n, f) != size_t(n)) return 6;
    mcsim::write_spikes_csv(argv[3], d);
  } else {
    mcsim::TraceData d;
    d.t_s = t;
    d.value.resize(n);
    if (n && std::fread(d.value.data(), 8, n, f) != size_t(n)) return 7;
    mcsim::write_trace_csv(argv[3], d);
  }
  std::fclose(f);
  return 0;
}
