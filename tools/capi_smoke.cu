// Standalone C-ABI smoke: no Python, no torch.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../include/eca_b200.h"
int main() {
  const int W = 320, H = 240, S = 16;
  std::vector<uint8_t> h(W * H * 3);
  for (int y = 0; y < H; ++y) for (int x = 0; x < W; ++x) {
    float dx = x - 159.5f, dy = y - 119.5f; uint8_t v = (dx*dx + dy*dy < 100.f*100.f) ? 150 : 3;
    for (int c = 0; c < 3; ++c) h[(y * W + x) * 3 + c] = v;
  }
  uint8_t* d; cudaMalloc(&d, h.size()); cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
  int32_t rows[S]; int n = eca_strip_rows(H, S, 8.0, rows); printf("rows %d\n", n); fflush(stdout);
  EcaParams p = {}; p.width = W; p.height = H; p.strip_count = 16; p.edge_margin_px = 3; p.ransac_attempts = 32; p.ransac_iterations = 3;
  p.gradient_threshold = 20; p.intensity_threshold = 25; p.angle_scale = 180.0 / (3.141592653589793 * 30.0);
  p.zero_grad_angle = 3.141592653589793 * p.angle_scale; p.min_point_score = 0.03; p.inlier_tol = 3.0 / W;
  p.circle_score_threshold = 0.96; p.min_radius_frac = 0.1; p.max_radius_frac = 0.8; p.max_center_offset_frac = 0.2;
  p.center_x = 159.5; p.center_y = 119.5;
  int32_t *x, *y; double* s; cudaMalloc(&x, 4 * 2 * n); cudaMalloc(&y, 4 * 2 * n); cudaMalloc(&s, 8 * 2 * n);
  printf("calling\n"); fflush(stdout);
  int rc = eca_points_handcrafted(d, 1, W * H * 3, W * 3, rows, nullptr, n, &p, x, y, s, nullptr);
  printf("rc %d\n", rc); fflush(stdout);
  cudaError_t e = cudaDeviceSynchronize(); printf("sync %s\n", cudaGetErrorString(e));
  std::vector<int32_t> hx(2 * n); cudaMemcpy(hx.data(), x, 4 * 2 * n, cudaMemcpyDeviceToHost);
  for (int i = 0; i < 2 * n; ++i) printf("%d ", hx[i]); printf("\n");
  return 0;
}
