// L1 gather micro-benchmark, 16 B records (float4), 128-bit loads.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__global__ void k(const float4 *data, const int *idx, int iters, int reps, float *out) {
    const int lane = threadIdx.x & 31;
    float acc = 0;
    for (int r = 0; r < reps; ++r)
        for (int it = 0; it < iters; it += 4) {
            int i0 = __ldg(idx + (it + 0) * 32 + lane), i1 = __ldg(idx + (it + 1) * 32 + lane);
            int i2 = __ldg(idx + (it + 2) * 32 + lane), i3 = __ldg(idx + (it + 3) * 32 + lane);
            float4 a = __ldg(data + i0), b = __ldg(data + i1), c = __ldg(data + i2), d = __ldg(data + i3);
            acc += a.x + b.y + c.z + d.w;
        }
    if (acc == 123.456f) out[0] = acc;
}
int main() {
    const int nrec = 2048;  // 32 KB
    const int iters = 64;
    std::vector<float4> h(nrec);
    for (int i = 0; i < nrec; ++i) h[i] = make_float4(i, 1, 2, 3);
    float4 *d; cudaMalloc(&d, nrec * sizeof(float4)); cudaMemcpy(d, h.data(), nrec * sizeof(float4), cudaMemcpyHostToDevice);
    float *out; cudaMalloc(&out, 8);
    int *di; cudaMalloc(&di, iters * 32 * 4);
    const char *names[] = {"coalesced", "8-lane groups: 8 consecutive (aligned 128 B)", "4-lane groups: 4 consecutive (aligned 64 B)",
                           "4-lane groups: same id mod 8 (stride 128 B)", "4-lane groups: 4*rand + s (distinct mod 4)",
                           "8-lane groups: 8*rand + s (distinct mod 8)", "random", "4-lane groups: 2*rand2 pairs (aligned 32 B pairs)",
                           "4-lane groups: 4 consecutive unaligned"};
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int pat = 0; pat < 9; ++pat) {
        std::vector<int> idx(iters * 32);
        srand(1);
        for (int it = 0; it < iters; ++it) {
            int r8[4], r4[8];
            for (int g = 0; g < 4; ++g) r8[g] = rand() % (nrec / 8);
            for (int g = 0; g < 8; ++g) r4[g] = rand() % (nrec / 4);
            for (int l = 0; l < 32; ++l) {
                int v = 0;
                switch (pat) {
                case 0: v = (it * 32 + l) % nrec; break;
                case 1: v = r8[l / 8] * 8 + l % 8; break;
                case 2: v = r4[l / 4] * 4 + l % 4; break;
                case 3: v = ((rand() % (nrec / 8)) * 8 + (l / 4)) % nrec; break;
                case 4: v = (rand() % (nrec / 4)) * 4 + l % 4; break;
                case 5: v = (rand() % (nrec / 8)) * 8 + l % 8; break;
                case 6: v = rand() % nrec; break;
                case 7: v = (l & 1) ? idx[it * 32 + l - 1] + 1 : (rand() % (nrec / 2)) * 2; break;
                case 8: v = (r4[l / 4] * 4 + 2 + l % 4) % nrec; break;
                }
                idx[it * 32 + l] = v;
            }
        }
        cudaMemcpy(di, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
        const int reps = 2000, blocks = sms * 4, threads = 256;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        k<<<blocks, threads>>>(d, di, iters, reps, out); cudaDeviceSynchronize();
        cudaEventRecord(e0); k<<<blocks, threads>>>(d, di, iters, reps, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double wl = (double)blocks * (threads / 32) * reps * iters / sms;
        double cyc = ms * 1e-3 * 1.965e9;
        printf("pat %d %-52s %.2f cyc per warp load per SM (incl. ~1 for the index load)\n", pat, names[pat], cyc / wl);
    }
    return 0;
}
