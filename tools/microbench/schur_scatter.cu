// Microbenchmark (tuning experiment, not product code): what bounds the Schur B^T scatter?
// Synthetic config-5-shaped B (nb rows x n cols, 2-4 random cols per row, SELL-32 by length).
//   A: t = Bv gathered, y[c] += b t by fp64 RED (the library's atomic form)
//   B: same, plain stores instead of RED (wrong result; cost of RED vs ST)
//   C: gather only, t written sequentially (cost of the v gather + B stream)
//   D: stream only (no gather: v[lane-local]) -> HBM floor for the B stream
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ss schur_scatter.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cmath>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) kb(const int* __restrict__ coff, const int* __restrict__ clen, int nch,
                                          const int* __restrict__ cols, const double* __restrict__ vals,
                                          const double* __restrict__ v, double* y, double* t) {
    const int lane = threadIdx.x & 31;
    const int ch = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (ch >= nch) return;
    const int len = clen[ch];
    const long long base = (long long)coff[ch] + lane;
    int c[4]; double b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) if (j < len) { c[j] = __ldcs(cols + base + 32LL * j); b[j] = __ldcs(vals + base + 32LL * j); }
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) if (j < len) acc += b[j] * (MODE == 3 ? v[(ch * 32 + lane) & 1023] : __ldg(v + c[j]));
    if (MODE == 0) {
#pragma unroll
        for (int j = 0; j < 4; ++j) if (j < len) atomicAdd(y + c[j], b[j] * acc);
    } else if (MODE == 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) if (j < len) y[c[j]] = b[j] * acc;
    } else {
        t[ch * 32 + lane] = acc;
    }
}


// ---- E: binned ("propagation blocking") form: phase 1 stages b*t per group of G_CH chunks in
// smem in bin order and writes one contiguous run per (group, bin); phase 2 accumulates one bin
// (a block of W columns) in smem.
constexpr int G_CH = 64;
__global__ void __launch_bounds__(256) kp1(const int* __restrict__ coff, const int* __restrict__ clen, int nch,
                                           const int* __restrict__ cols, const double* __restrict__ vals,
                                           const unsigned short* __restrict__ lpos, const double* __restrict__ v,
                                           const int* __restrict__ RS, const int* __restrict__ O, int nbins,
                                           double* __restrict__ bins) {
    extern __shared__ double stage[];
    int* srs = reinterpret_cast<int*>(stage + G_CH * 32 * 4);
    int* so = srs + nbins + 1;
    const int g = blockIdx.x;
    for (int p = threadIdx.x; p <= nbins; p += blockDim.x) {
        srs[p] = RS[(size_t)g * (nbins + 1) + p];
        if (p < nbins) so[p] = O[(size_t)g * nbins + p];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ch0 = g * G_CH, ch1 = min(nch, ch0 + G_CH);
    const int gbase = coff[ch0];
    for (int ch = ch0 + warp; ch < ch1; ch += 8) {
        const int len = clen[ch];
        const long long base = (long long)coff[ch] + lane;
        int c[4]; double b[4]; int lp[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) if (j < len) { c[j] = __ldcs(cols + base + 32LL * j); b[j] = __ldcs(vals + base + 32LL * j); lp[j] = lpos[base + 32LL * j]; }
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 4; ++j) if (j < len) acc += b[j] * __ldg(v + c[j]);
#pragma unroll
        for (int j = 0; j < 4; ++j) if (j < len) stage[lp[j]] = b[j] * acc;
    }
    (void)gbase;
    __syncthreads();
    for (int p = warp; p < nbins; p += 8) {
        const int r0 = srs[p], L = srs[p + 1] - r0;
        double* dst = bins + so[p];
        for (int k = lane; k < L; k += 32) __stcg(dst + k, stage[r0 + k]);
    }
}

__global__ void __launch_bounds__(512) kp2(const int* __restrict__ binstart, const unsigned short* __restrict__ colloc,
                                           const double* __restrict__ bins, int W, int n, double* __restrict__ y) {
    extern __shared__ double sy[];
    const int p = blockIdx.x;
    const int c0 = p * W, w = min(W, n - c0);
    for (int i = threadIdx.x; i < w; i += blockDim.x) sy[i] = 0.0;
    __syncthreads();
    const int e0 = binstart[p], e1 = binstart[p + 1];
    for (int e = e0 + threadIdx.x; e < e1; e += blockDim.x) atomicAdd(&sy[colloc[e]], __ldcs(bins + e));
    __syncthreads();
    for (int i = threadIdx.x; i < w; i += blockDim.x) y[c0 + i] = sy[i];
}

int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 4000000;
    const int nb = 3 * n;
    std::mt19937_64 g(4);
    std::vector<int> len(nb);
    for (auto& l : len) l = 2 + (int)(g() % 3);
    std::vector<int> order(nb);
    for (int i = 0; i < nb; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return len[a] > len[b]; });
    std::vector<int> coff{0}, clen;
    for (int i = 0; i < nb; i += 32) {
        int L = 0;
        for (int l = 0; l < 32 && i + l < nb; ++l) L = std::max(L, len[order[i + l]]);
        clen.push_back(L);
        coff.push_back(coff.back() + 32 * L);
    }
    const int nch = (int)clen.size();
    std::vector<int> cols(coff.back());
    std::vector<double> vals(coff.back());
    for (int ch = 0; ch < nch; ++ch)
        for (int l = 0; l < 32; ++l)
            for (int j = 0; j < clen[ch]; ++j) {
                cols[coff[ch] + 32 * j + l] = (int)(g() % n);
                vals[coff[ch] + 32 * j + l] = 1.0;
            }
    int *dcoff, *dclen, *dcols; double *dvals, *dv, *dy, *dt;
    cudaMalloc(&dcoff, 4 * coff.size()); cudaMalloc(&dclen, 4 * clen.size());
    cudaMalloc(&dcols, 4 * cols.size()); cudaMalloc(&dvals, 8 * vals.size());
    cudaMalloc(&dv, 8 * (size_t)n); cudaMalloc(&dy, 8 * (size_t)n); cudaMalloc(&dt, 8 * (size_t)nb + 1024);
    cudaMemcpy(dcoff, coff.data(), 4 * coff.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dclen, clen.data(), 4 * clen.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dcols, cols.data(), 4 * cols.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dvals, vals.data(), 8 * vals.size(), cudaMemcpyHostToDevice);
    cudaMemset(dv, 0, 8 * (size_t)n); cudaMemset(dy, 0, 8 * (size_t)n);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const char* names[] = {"A atomic RED", "B plain ST", "C gather only", "D stream only"};
    const double slots = (double)coff.back();
    for (int mode = 0; mode < 4; ++mode) {
        auto run = [&]() {
            dim3 gr((nch + 7) / 8);
            if (mode == 0) kb<0><<<gr, 256>>>(dcoff, dclen, nch, dcols, dvals, dv, dy, dt);
            if (mode == 1) kb<1><<<gr, 256>>>(dcoff, dclen, nch, dcols, dvals, dv, dy, dt);
            if (mode == 2) kb<2><<<gr, 256>>>(dcoff, dclen, nch, dcols, dvals, dv, dy, dt);
            if (mode == 3) kb<3><<<gr, 256>>>(dcoff, dclen, nch, dcols, dvals, dv, dy, dt);
        };
        for (int i = 0; i < 3; ++i) run();
        cudaEventRecord(e0);
        for (int i = 0; i < 20; ++i) run();
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
        printf("%-16s %8.1f us  %6.2f Gslot/s  stream %6.0f GB/s  err=%s\n", names[mode], ms * 1e3, slots / (ms * 1e6),
               slots * 12 / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
    }

    // ---------------- E: binned form
    {
        const int nbins = argc > 2 ? atoi(argv[2]) : 296;
        const int W = (n + nbins - 1) / nbins;
        const int G = (nch + G_CH - 1) / G_CH;
        std::vector<int> RS((size_t)G * (nbins + 1)), O((size_t)G * nbins), cnt((size_t)G * nbins, 0);
        std::vector<unsigned short> lpos(coff.back());
        std::vector<long long> bintot(nbins, 0);
        for (int gi = 0; gi < G; ++gi) {
            const int s0 = coff[gi * G_CH], s1 = coff[std::min(nch, (gi + 1) * G_CH)];
            for (int s = s0; s < s1; ++s) cnt[(size_t)gi * nbins + cols[s] / W]++;
            int acc = 0;
            for (int p = 0; p < nbins; ++p) { RS[(size_t)gi * (nbins + 1) + p] = acc; acc += cnt[(size_t)gi * nbins + p]; bintot[p] += cnt[(size_t)gi * nbins + p]; }
            RS[(size_t)gi * (nbins + 1) + nbins] = acc;
            std::vector<int> fill(nbins, 0);
            for (int s = s0; s < s1; ++s) { int p = cols[s] / W; lpos[s] = (unsigned short)(RS[(size_t)gi * (nbins + 1) + p] + fill[p]++); }
        }
        std::vector<int> binstart(nbins + 1, 0);
        for (int p = 0; p < nbins; ++p) binstart[p + 1] = binstart[p] + (int)bintot[p];
        std::vector<int> run(nbins, 0);
        std::vector<unsigned short> colloc(coff.back());
        for (int gi = 0; gi < G; ++gi)
            for (int p = 0; p < nbins; ++p) {
                O[(size_t)gi * nbins + p] = binstart[p] + run[p];
                run[p] += cnt[(size_t)gi * nbins + p];
            }
        for (int gi = 0; gi < G; ++gi) {
            const int s0 = coff[gi * G_CH], s1 = coff[std::min(nch, (gi + 1) * G_CH)];
            for (int s = s0; s < s1; ++s) {
                int p = cols[s] / W;
                int k = lpos[s] - RS[(size_t)gi * (nbins + 1) + p];
                colloc[O[(size_t)gi * nbins + p] + k] = (unsigned short)(cols[s] - p * W);
            }
        }
        unsigned short *dlpos, *dcolloc; int *dRS, *dO, *dbs; double *dbins, *dy2;
        cudaMalloc(&dlpos, 2 * lpos.size()); cudaMalloc(&dcolloc, 2 * colloc.size());
        cudaMalloc(&dRS, 4 * RS.size()); cudaMalloc(&dO, 4 * O.size()); cudaMalloc(&dbs, 4 * binstart.size());
        cudaMalloc(&dbins, 8 * (size_t)coff.back()); cudaMalloc(&dy2, 8 * (size_t)n);
        cudaMemcpy(dlpos, lpos.data(), 2 * lpos.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dcolloc, colloc.data(), 2 * colloc.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dRS, RS.data(), 4 * RS.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dO, O.data(), 4 * O.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dbs, binstart.data(), 4 * binstart.size(), cudaMemcpyHostToDevice);
        // random v for a correctness check against the atomic form
        std::vector<double> hv(n);
        for (auto& x : hv) x = (double)(g() % 1000) / 1000.0 - 0.5;
        cudaMemcpy(dv, hv.data(), 8 * (size_t)n, cudaMemcpyHostToDevice);
        cudaMemset(dy, 0, 8 * (size_t)n);
        kb<0><<<(nch + 7) / 8, 256>>>(dcoff, dclen, nch, dcols, dvals, dv, dy, dt);
        const size_t sm1 = 8 * G_CH * 32 * 4 + 4 * (2 * nbins + 1);
        const size_t sm2 = 8 * (size_t)W;
        cudaFuncSetAttribute(kp1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
        cudaFuncSetAttribute(kp2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
        auto p1 = [&]() { kp1<<<G, 256, sm1>>>(dcoff, dclen, nch, dcols, dvals, dlpos, dv, dRS, dO, nbins, dbins); };
        auto p2 = [&]() { kp2<<<nbins, 512, sm2>>>(dbs, dcolloc, dbins, W, n, dy2); };
        p1(); p2(); cudaDeviceSynchronize();
        std::vector<double> ya(n), yb(n);
        cudaMemcpy(ya.data(), dy, 8 * (size_t)n, cudaMemcpyDeviceToHost);
        cudaMemcpy(yb.data(), dy2, 8 * (size_t)n, cudaMemcpyDeviceToHost);
        double md = 0, mx = 0;
        for (int i = 0; i < n; ++i) { md = std::max(md, std::abs(ya[i] - yb[i])); mx = std::max(mx, std::abs(ya[i])); }
        printf("E check: max|y_atomic - y_binned| = %.3e (max|y| %.3e) err=%s\n", md, mx, cudaGetErrorString(cudaGetLastError()));
        for (int which = 0; which < 3; ++which) {
            for (int i = 0; i < 3; ++i) { if (which != 1) p1(); if (which != 0) p2(); }
            cudaEventRecord(e0);
            for (int i = 0; i < 20; ++i) { if (which != 1) p1(); if (which != 0) p2(); }
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
            const char* nm[] = {"E phase1", "E phase2", "E total"};
            printf("%-16s %8.1f us  nbins %d W %d G %d smem %zu/%zu\n", nm[which], ms * 1e3, nbins, W, G, sm1, sm2);
        }
    }
    return 0;
}
