// C++ performance leg: configs 1-4 through the drop-in headers
// (tiletensor_b200/*.hpp -- the reference's own tiletensor:: API, bodies on the
// C-ABI), timed per call from the host exactly as a C++ caller of the
// reference would use it.  Each call allocates its result from the session's
// stream-ordered pool (tt_device_alloc) and enqueues its kernels on the
// session stream; the loop is drained once at the end, so the per-call time
// is max(host enqueue cost, device time).  Prints one JSON object.
//
// Inputs are seeded uniform draws (the timings do not depend on values;
// parity of these paths is covered by tests_cpp/host_tests.cpp and the
// Python suite).  Build: paper_2011_01805_b200/build.py (build_cpp_bench).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

// the reference's own include names (proj/include/tiletensor/*.hpp), resolved to
// the drop-in headers by paper_2011_01805_b200/include/tiletensor/
#include "tiletensor/linalg.hpp"
#include "tiletensor/tile_tensor.hpp"

using namespace tiletensor;
using clk = std::chrono::steady_clock;

static DenseTensor uniform(std::vector<std::int64_t> shape, std::uint64_t seed, double lo = -1, double hi = 1) {
  std::int64_t n = 1;
  for (auto e : shape) n *= e;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(lo, hi);
  std::vector<double> v(static_cast<std::size_t>(n));
  for (auto& x : v) x = u(rng);
  return DenseTensor(std::move(shape), std::move(v));
}

// Mean seconds per call of `fn` over `reps` calls after `warm` warm-up calls,
// the session stream drained before and after.
static double per_call(Session& s, int warm, int reps, const std::function<void()>& fn) {
  for (int i = 0; i < warm; ++i) fn();
  detail::check(tt_session_synchronize(s.handle()));
  const auto t0 = clk::now();
  for (int i = 0; i < reps; ++i) fn();
  detail::check(tt_session_synchronize(s.handle()));
  return std::chrono::duration<double>(clk::now() - t0).count() / reps;
}

// The same call captured once into a CUDA graph on the session stream and
// replayed: the device-side floor of the call without host launch cost.
static double graph_replay(Session& s, int reps, const std::function<void()>& fn) {
  cudaStream_t st = static_cast<cudaStream_t>(tt_session_stream(s.handle()));
  for (int i = 0; i < 3; ++i) fn();
  detail::check(tt_session_synchronize(s.handle()));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  if (cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return -1;
  fn();
  if (cudaStreamEndCapture(st, &g) != cudaSuccess) return -1;
  if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) return -1;
  cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  const auto t0 = clk::now();
  for (int i = 0; i < reps; ++i) cudaGraphLaunch(ge, st);
  cudaStreamSynchronize(st);
  const double t = std::chrono::duration<double>(clk::now() - t0).count() / reps;
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return t;
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? std::atoi(argv[1]) : 200;
  std::string json = "{";
  auto emit = [&](const char* name, double call, double graph) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "%s\"%s\": {\"us\": %.3f, \"graph_replay_us\": %.3f}",
                  json.size() > 1 ? ", " : "", name, call * 1e6, graph * 1e6);
    json += buf;
  };
  {  // config 1: tt_sum(tt_mul(A, B), 2) fused, [100/16,200/32], 512 slots
    Session s(512, 8);
    const auto sh = parse_shape("[100/16,200/32]");
    const TileTensor a = pack(uniform({100, 200}, 1), sh, s), b = pack(uniform({100, 200}, 2), sh, s);
    auto f = [&] { (void)tt_mul_sum(a, b, 2); };
    emit("c1_mul_sum", per_call(s, 50, reps * 10, f), graph_replay(s, reps * 10, f));
  }
  {  // config 2: matvec_a(M [1024/64,4096/128], V [*/64,4096/128])
    Session s(8192, 8);
    const TileTensor m = pack(uniform({1024, 4096}, 3), parse_shape("[1024/64,4096/128]"), s);
    const TileTensor v = pack(uniform({1, 4096}, 4), parse_shape("[*/64,4096/128]"), s);
    auto f = [&] { (void)matvec_a(m, v); };
    emit("c2_matvec", per_call(s, 20, reps * 4, f), graph_replay(s, reps * 4, f));
  }
  {  // config 3 "3b": matmul_a(A, matmul_b(Bt, C))
    Session s(8192, 8);
    const TileTensor a = pack(uniform({512, 1024, 1}, 5), parse_shape("[512/16,1024/32,*/16]"), s);
    const TileTensor bt = pack(uniform({768, 1024, 1}, 6), parse_shape("[768/16,1024/32,*/16]"), s);
    const TileTensor c = pack(uniform({768, 1, 256}, 7), parse_shape("[768/16,*/32,256/16]"), s);
    auto f = [&] { (void)matmul_a(a, matmul_b(bt, c)); };
    emit("c3b_matmul_chain", per_call(s, 5, reps, f), graph_replay(s, reps, f));
  }
  {  // config 4: FC 784->100 + bias + square, FC 100->10 + bias (tt_mul_sum_affine per layer)
    Session s(8192, 8);
    const TileTensor x = pack(uniform({784, 1, 4096}, 8, 0, 1), parse_shape("[784/32,1,4096~/256]"), s);
    const TileTensor w1 = pack(uniform({784, 100, 1}, 9), parse_shape("[784/32,100,*/256]"), s);
    const TileTensor b1 = pack(uniform({1, 100, 1}, 11), parse_shape("[*/32,100,*/256]"), s);
    const TileTensor w2 = pack(uniform({10, 100, 1}, 10), parse_shape("[10/32,100,*/256]"), s);
    const TileTensor b2 = pack(uniform({10, 1, 1}, 12), parse_shape("[10/32,1,*/256]"), s);
    auto f = [&] {
      const TileTensor h = tt_mul_sum_affine(w1, x, 1, &b1, true);
      (void)tt_mul_sum_affine(w2, h, 2, &b2, false);
    };
    emit("c4_fc_square_fc", per_call(s, 5, reps, f), graph_replay(s, reps, f));
  }
  json += "}";
  std::printf("%s\n", json.c_str());
  return 0;
}
