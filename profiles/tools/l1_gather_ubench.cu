// L1 gather micro-benchmark: cycles per warp-wide 256-bit load for several lane->record patterns.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ double4 ldg4(const double4 *p) {
    double4 v;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
// idx: [iters][32] record ids (within a region of nrec records)
template <int W>
__global__ void k(const double4 *data, const int *idx, int iters, int reps, double *out) {
    const int lane = threadIdx.x & 31;
    double acc = 0;
    for (int r = 0; r < reps; ++r)
        for (int it = 0; it < iters; it += 4) {
            int i0 = __ldg(idx + (it + 0) * 32 + lane), i1 = __ldg(idx + (it + 1) * 32 + lane);
            int i2 = __ldg(idx + (it + 2) * 32 + lane), i3 = __ldg(idx + (it + 3) * 32 + lane);
            if (W == 32) {
                double4 a = ldg4(data + i0), b = ldg4(data + i1), c = ldg4(data + i2), d = ldg4(data + i3);
                acc += a.x + b.y + c.z + d.w;
            } else if (W == 16) {
                const double2 *p = reinterpret_cast<const double2 *>(data);
                double2 a = __ldg(p + 2 * i0), b = __ldg(p + 2 * i1), c = __ldg(p + 2 * i2), d = __ldg(p + 2 * i3);
                acc += a.x + b.y + c.x + d.y;
            } else {
                const double *p = reinterpret_cast<const double *>(data);
                acc += __ldg(p + 4 * i0) + __ldg(p + 4 * i1) + __ldg(p + 4 * i2) + __ldg(p + 4 * i3);
            }
        }
    if (acc == 123.456) out[0] = acc;
}
int main() {
    const int nrec = 1024;  // 32 KB region: L1 resident
    const int iters = 64;
    std::vector<double4> h(nrec);
    for (int i = 0; i < nrec; ++i) h[i] = make_double4(i, 1, 2, 3);
    double4 *d; cudaMalloc(&d, nrec * sizeof(double4)); cudaMemcpy(d, h.data(), nrec * sizeof(double4), cudaMemcpyHostToDevice);
    double *out; cudaMalloc(&out, 8);
    int *di; cudaMalloc(&di, iters * 32 * 4);
    const char *names[] = {"coalesced (8 full lines)", "8 random aligned quads", "quads straddling 2 lines (16 touches)",
                           "32 random records (32 lines)", "all lanes same record", "4-lane groups: same record per group",
                           "pairs: 16 random aligned pairs (16 lines)", "8 random lines, lanes permuted across groups",
                           "32 random lines, offset = lane % 4 (bank-balanced groups)", "16 random lines: group = 2 lines x 2 records, offsets distinct", "32 random lines, offsets = 2 x {0,1} per group (2-way)"};
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int pat = 0; pat < 11; ++pat) {
        std::vector<int> idx(iters * 32);
        srand(1);
        for (int it = 0; it < iters; ++it) {
            int quad[8]; for (int g = 0; g < 8; ++g) quad[g] = rand() % (nrec / 4);
            for (int l = 0; l < 32; ++l) {
                int g = l / 4, s = l % 4, v = 0;
                switch (pat) {
                case 0: v = (it * 32 + l) % nrec; break;
                case 1: v = quad[g] * 4 + s; break;
                case 2: v = (quad[g] * 4 + 2 + s) % nrec; break;
                case 3: v = rand() % nrec; break;
                case 4: v = quad[0] * 4; break;
                case 5: v = quad[g] * 4; break;
                case 6: v = ((rand() % (nrec / 2)) * 2 * ((l & 1) == 0) + 0); if (l & 1) v = idx[it * 32 + l - 1] + 1; break;
                case 7: v = quad[l % 8] * 4 + (l / 8); break;
                case 8: v = (rand() % (nrec / 4)) * 4 + s; break;
                case 9: v = (s & 1) ? idx[it * 32 + l - 1] + 1 : (rand() % (nrec / 4)) * 4 + s; break;
                case 10: v = (rand() % (nrec / 4)) * 4 + (s & 1); break;
                }
                idx[it * 32 + l] = v;
            }
        }
        cudaMemcpy(di, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
        for (int W : {32, 16, 8}) {
            const int reps = 2000, blocks = sms * 4, threads = 256;
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            auto run = [&]() {
                if (W == 32) k<32><<<blocks, threads>>>(d, di, iters, reps, out);
                else if (W == 16) k<16><<<blocks, threads>>>(d, di, iters, reps, out);
                else k<8><<<blocks, threads>>>(d, di, iters, reps, out);
            };
            run(); cudaDeviceSynchronize();
            cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            double warp_loads_per_sm = (double)blocks * (threads / 32) * reps * iters / sms;
            double cyc = ms * 1e-3 * 1.965e9;  // at max clock
            printf("pat %d %-48s W=%2d B: %.2f cyc per warp load per SM (%.1f B/clk/SM)\n", pat, names[pat], W,
                   cyc / warp_loads_per_sm, warp_loads_per_sm * 32 * W / cyc);
        }
    }
    return 0;
}
