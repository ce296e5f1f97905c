// C++ host-side parity driver (test infrastructure): drives the B200 decode
// path through include/thinkv_b200.hpp exactly as a C++ caller of the
// reference would drive ThinkvMethod (proj/src/sim.cpp:748-843), on the
// golden walkthrough of proj/tests/test_sim.cpp:386-489 (tau = g = block = 4,
// schedule {2}, scripted R,E,T,R).  Inputs (fp64 q/k/v per step) are read
// from argv[1]; the step dumps are written to stdout as JSON.  With argv[2]
// == "oom" it instead checks that pool exhaustion surfaces as
// thinkv_b200::Error with exit_code() 4 (pager.cpp:29-37, errors.hpp:31-46).
#include <cstdio>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

#include "thinkv_b200.hpp"

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s inputs.f64 [oom]\n", argv[0]);
    return 2;
  }
  using thinkv_b200::Context;
  using thinkv_b200::DecodeRun;
  const bool oom = argc > 2 && std::strcmp(argv[2], "oom") == 0;
  constexpr int kSteps = 16, kD = 4;
  std::vector<double> in(3 * kSteps * kD);
  if (!oom) {
    FILE* f = std::fopen(argv[1], "rb");
    if (!f || std::fread(in.data(), sizeof(double), in.size(), f) != in.size()) {
      std::fprintf(stderr, "cannot read %s\n", argv[1]);
      return 2;
    }
    std::fclose(f);
  }
  tkv_run_desc d{};
  d.num_seqs = 1; d.units_per_seq = 1; d.num_q_heads = 1; d.head_dim = kD;
  d.tau = 4; d.group_size = 4; d.block_size = 4; d.pool_blocks = oom ? 2 : 16;
  d.budget = oom ? 4096 : 64; d.num_levels = 1; d.levels[0] = 2;
  d.psi_bits[0] = 4; d.psi_bits[1] = 4; d.psi_bits[2] = 2;  // E, R, T
  d.num_thoughts = 3; d.threshold_fraction = 0.01; d.max_gen_len = kSteps;
  const int32_t script[4] = {1, 0, 2, 1};  // R, E, T, R
  d.scripted = 1; d.script_len = 4; d.script_bands = script;
  d.input_dtype = TKV_DTYPE_F64; d.record_events = 1;
  const int64_t dumps[5] = {3, 7, 11, 12, 15};
  d.num_dump_positions = oom ? 0 : 5; d.dump_positions = dumps;

  Context ctx(0);
  DecodeRun run(ctx, d);
  double *q, *k, *v;
  float* out;
  cudaMalloc(&q, kD * sizeof(double));
  cudaMalloc(&k, kD * sizeof(double));
  cudaMalloc(&v, kD * sizeof(double));
  cudaMalloc(&out, kD * sizeof(float));
  try {
    for (int t = 0; t < kSteps; ++t) {
      cudaMemcpy(q, &in[(0 * kSteps + t) * kD], kD * sizeof(double), cudaMemcpyHostToDevice);
      cudaMemcpy(k, &in[(1 * kSteps + t) * kD], kD * sizeof(double), cudaMemcpyHostToDevice);
      cudaMemcpy(v, &in[(2 * kSteps + t) * kD], kD * sizeof(double), cudaMemcpyHostToDevice);
      run.process(q, k, v, out);
    }
    run.finish();
  } catch (const thinkv_b200::Error& e) {
    if (oom && e.exit_code() == 4) {
      std::printf("{\"oom_exit_code\": %d}\n", e.exit_code());
      return 0;
    }
    std::fprintf(stderr, "error %d: %s\n", e.exit_code(), e.what());
    return e.exit_code();
  }
  if (oom) {
    std::fprintf(stderr, "expected an out-of-memory error\n");
    return 1;
  }
  std::printf("%s\n", run.dump("step_dumps").c_str());
  return 0;
}
