// Stand-alone timing of the fused smoother chain (chain.cuh) on a synthetic
// level-9-like A_ff (rows x ~len entries in a band), with a per-CTA
// %globaltimer trace of its phases.  nvcc -arch=sm_100a -O3 -I.. chain_bench.cu
#define CHAIN_TRACE 1
#include "../../paper_2508_17517_b200/csrc/chain.cuh"
#include <cstdio>
#include <vector>
#include <random>
#include <algorithm>
#include <string>
using namespace airg;
void set_error(const char*, ...) {}
namespace airg { void set_error(const char*, ...) {} }

template <int VS>
__global__ void spmv_step(int n, const int* ptr, const int* col, const double* val, const double* x,
                          double xs, const double* b, double cj, double* y) {
  const int lane = threadIdx.x & (VS - 1);
  const long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / VS;
  double s = 0;
  if (row < n) s = chain_row<VS, false>(col, val, ptr[row], ptr[row + 1], lane, x, xs);
  else s = chain_row<VS, false>(col, val, 0, 0, lane, x, xs);
  if (row < n && lane == 0) y[row] = fma(cj, b[row], s);
}

int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 14133;
  const int len = argc > 2 ? atoi(argv[2]) : 155;
  const int G = argc > 3 ? atoi(argv[3]) : 148;
  const int d = 6;
  std::mt19937 rng(1);
  std::vector<int> ptr(n + 1), col;
  std::vector<double> val;
  if (argc > 4) {  // real matrix: <prefix>_ptr.bin / _col.bin / _val.bin
    auto rd = [](const std::string& f, auto& v) {
      FILE* fp = fopen(f.c_str(), "rb");
      fseek(fp, 0, SEEK_END); long sz = ftell(fp); fseek(fp, 0, SEEK_SET);
      v.resize(sz / sizeof(v[0])); fread(v.data(), 1, sz, fp); fclose(fp);
    };
    rd(std::string(argv[4]) + "_ptr.bin", ptr);
    rd(std::string(argv[4]) + "_col.bin", col);
    rd(std::string(argv[4]) + "_val.bin", val);
  }
  const int nreal = argc > 4 ? (int)ptr.size() - 1 : n;
  for (int i = 0; i < n && argc <= 4; ++i) {
    ptr[i] = (int)col.size();
    int L = std::max(1, (int)(len * (0.7 + 0.6 * (rng() % 1000) / 1000.0)));
    std::vector<int> c;
    for (int k = 0; k < L; ++k) c.push_back(std::min(n - 1, std::max(0, i + (int)(rng() % 2001) - 1000)));
    std::sort(c.begin(), c.end());
    c.erase(std::unique(c.begin(), c.end()), c.end());
    for (int x : c) { col.push_back(x); val.push_back(1e-3 * ((int)(rng() % 2001) - 1000)); }
  }
  if (argc <= 4) ptr[n] = (int)col.size();
  n = nreal;
  const long long nnz = col.size();
  int *dp, *dc, *part; double *dv, *b, *t0, *t1, *y, *y2; unsigned long long* bar; long long* trace;
  cudaMalloc(&dp, 4 * (n + 1)); cudaMalloc(&dc, 4 * nnz); cudaMalloc(&dv, 8 * nnz);
  cudaMalloc(&b, 8 * n); cudaMalloc(&t0, 8 * n); cudaMalloc(&t1, 8 * n); cudaMalloc(&y, 8 * n); cudaMalloc(&y2, 8 * n);
  cudaMalloc(&part, 12 * G + 4); cudaMemset(part, 0, 12 * G + 4); cudaMalloc(&bar, 8); cudaMemset(bar, 0, 8);
  const int NT = 4 + 2 * d;
  cudaMalloc(&trace, 8 * G * NT);
  cudaMemcpy(dp, ptr.data(), 4 * (n + 1), cudaMemcpyHostToDevice);
  cudaMemcpy(dc, col.data(), 4 * nnz, cudaMemcpyHostToDevice);
  cudaMemcpy(dv, val.data(), 8 * nnz, cudaMemcpyHostToDevice);
  std::vector<double> hb(n); for (auto& x : hb) x = (rng() % 1000) / 1000.0;
  cudaMemcpy(b, hb.data(), 8 * n, cudaMemcpyHostToDevice);
  int optin; cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  const int smem = optin - 1024;
  long long* wbuf; cudaMalloc(&wbuf, 8 * (n + 1));
  const int vs = argc > 5 ? atoi(argv[5]) : 32;
  {  // exclusive prefix of the row costs on the host (test harness)
    std::vector<long long> w(n + 1, 0);
    const int step = kChainU * vs;
    for (int i = 0; i < n; ++i) w[i + 1] = w[i] + (long long)((ptr[i + 1] - ptr[i] + step - 1) / step) * step + 4;
    cudaMemcpy(wbuf, w.data(), 8 * (n + 1), cudaMemcpyHostToDevice);
  }
  chain_partition_kernel<<<(G + 127) / 128, 128>>>(n, dp, G, smem - 128, wbuf, part);
  int need = 0;
  cudaMemcpy(&need, part + 3 * G, 4, cudaMemcpyDeviceToHost);
  const int lsmem = argc > 6 && atoi(argv[6]) ? std::min(smem, ((need + 1023) / 1024) * 1024 + 1024) : smem;
  printf("staged bytes max %d, launch smem %d\n", need, lsmem);
  ChainArgs a{};
  a.n = n; a.ptr = dp; a.col = dc; a.val = dv; a.b = b; a.t0 = t0; a.t1 = t1; a.y = y; a.ymap = nullptr;
  a.part = part; a.bar = bar; a.d = d; a.smem = lsmem; a.trace = trace;
  for (int j = 0; j <= d; ++j) a.coef[j] = 0.5 + 0.1 * j;
  cudaFuncSetAttribute(chain_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G); cfg.blockDim = dim3(kChainThreads); cfg.dynamicSmemBytes = lsmem;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) cudaLaunchKernelEx(&cfg, chain_kernel<32>, a);
  cudaEventRecord(e0);
  const int R = 20;
  for (int w = 0; w < R; ++w) cudaLaunchKernelEx(&cfg, chain_kernel<32>, a);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("chain: %.1f us per launch (n %d nnz %lld, G %d) err=%s\n", ms * 1000 / R, n, nnz, G,
         cudaGetErrorString(cudaGetLastError()));
  // multi-launch reference
  const int blocks = (int)(((long long)n * 32 + 255) / 256);
  auto multi = [&]() {
    const double* x = b; double xs = a.coef[d];
    for (int j = d - 1; j >= 0; --j) {
      double* dst = j == 0 ? y2 : ((j & 1) ? t1 : t0);
      spmv_step<32><<<blocks, 256>>>(n, dp, dc, dv, x, xs, b, a.coef[j], dst);
      x = dst; xs = 1.0;
    }
  };
  for (int w = 0; w < 3; ++w) multi();
  cudaEventRecord(e0);
  for (int w = 0; w < R; ++w) multi();
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("multi: %.1f us per %d launches\n", ms * 1000 / R, d);
  std::vector<double> h1(n), h2(n);
  cudaMemcpy(h1.data(), y, 8 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), y2, 8 * n, cudaMemcpyDeviceToHost);
  double md = 0, mx = 0;
  for (int i = 0; i < n; ++i) { md = std::max(md, fabs(h1[i] - h2[i])); mx = std::max(mx, fabs(h2[i])); }
  printf("max diff %.3e (max %.3e)\n", md, mx);
  // trace of the last launch
  std::vector<long long> tr(G * NT);
  cudaMemcpy(tr.data(), trace, 8 * G * NT, cudaMemcpyDeviceToHost);
  long long t00 = tr[0];
  for (int g = 0; g < G; ++g) t00 = std::min(t00, tr[g * NT]);
  for (int p = 0; p < NT; ++p) {
    long long lo = 1LL << 62, hi = 0; double avg = 0;
    for (int g = 0; g < G; ++g) { long long v = tr[g * NT + p] - t00; lo = std::min(lo, v); hi = std::max(hi, v); avg += v; }
    printf("point %2d: min %7.2f avg %7.2f max %7.2f us\n", p, lo / 1e3, avg / G / 1e3, hi / 1e3);
  }
  // slowest CTAs of step 1 (arrival - release of step 0) and their blocks
  std::vector<int> hp(3 * G);
  cudaMemcpy(hp.data(), part, 12 * G, cudaMemcpyDeviceToHost);
  std::vector<std::pair<long long, int>> dur;
  for (int g = 0; g < G; ++g) dur.push_back({tr[g * NT + 5] - tr[g * NT + 4], g});
  std::sort(dur.rbegin(), dur.rend());
  for (int q = 0; q < 6 && q < G; ++q) {
    const int g = dur[q].second, r0 = hp[3 * g], rs = hp[3 * g + 1], r1 = hp[3 * g + 2];
    long long nz = ptr[r1] - ptr[r0], spread = 0, maxspan = 0;
    for (int i = r0; i < r1; ++i) {
      if (ptr[i + 1] > ptr[i]) {
        spread += col[ptr[i + 1] - 1] - col[ptr[i]];
        maxspan = std::max<long long>(maxspan, col[ptr[i + 1] - 1] - col[ptr[i]]);
      }
    }
    printf("cta %3d: step1 %.2f us rows [%d,%d) staged to %d nnz %lld mean col span %.0f max %lld\n", g,
           dur[q].first / 1e3, r0, r1, rs, nz, r1 > r0 ? (double)spread / (r1 - r0) : 0.0, maxspan);
  }
  const int g = dur[G / 2].second;
  printf("median cta %d: %.2f us rows [%d,%d) staged to %d\n", g, dur[G / 2].first / 1e3, hp[3 * g],
         hp[3 * g + 2], hp[3 * g + 1]);
  return 0;
}
