// Host-side profile target: config 1's fused op through the C-ABI in a loop
// (gprofng collect app ./capi_loop).  Build:
// g++ -O2 -g -I include -o tools/micro/capi_loop tools/micro/capi_loop.cpp -Lpaper_2011_01805_b200/_lib -ltiletensor_b200 -Wl,-rpath,$PWD/paper_2011_01805_b200/_lib
#include <chrono>
#include <cstdio>
#include <vector>
#include "tiletensor_b200.h"
int main() {
  tt_session* s;
  if (tt_session_create(512, 8, 0, &s)) return 1;
  tt_shape sh;
  tt_shape_parse("[100/16,200/32]", &sh);
  void *a, *b, *o;
  tt_device_alloc(s, 49 * 512 * 8, &a);
  tt_device_alloc(s, 49 * 512 * 8, &b);
  tt_device_alloc(s, 7 * 512 * 8, &o);
  tt_session_synchronize(s);
  for (int pass = 0; pass < 2; ++pass) {
    const int n = pass ? 200000 : 1000;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i)
      tt_mul_sum(s, &sh, (double*)a, 8, &sh, (double*)b, 8, 2, -1, nullptr, (double*)o, nullptr);
    tt_session_synchronize(s);
    auto t1 = std::chrono::steady_clock::now();
    if (pass) printf("tt_mul_sum c1: %.2f us/call\n", std::chrono::duration<double>(t1 - t0).count() / n * 1e6);
  }
  return 0;
}
