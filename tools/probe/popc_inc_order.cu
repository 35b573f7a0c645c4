// Probe: does atomicAdd(&smem[d], 1) (ATOMS.POPC.INC) hand out per-address
// values in ascending lane order? Counts violations over many random patterns.
#include <cstdio>
#include <cstdint>
__global__ void probe(int iters, unsigned long long* bad, unsigned long long* total, int bins) {
    __shared__ uint32_t cnt[8][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t x = 0x9E3779B9u * (blockIdx.x * blockDim.x + threadIdx.x + 1);
    unsigned long long nb = 0, nt = 0;
    for (int it = 0; it < iters; ++it) {
        for (int i = lane; i < 256; i += 32) cnt[warp][i] = 0;
        __syncwarp();
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        const uint32_t d = (x >> 8) % bins;
        const uint32_t r = atomicAdd(&cnt[warp][d], 1u);
        // lanes with the same digit must get increasing values by lane
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        const uint32_t below = __popc(peers & ((1u << lane) - 1));
        nb += (r != below);
        nt += 1;
        __syncwarp();
    }
    atomicAdd(bad, nb);
    atomicAdd(total, nt);
}
int main() {
    unsigned long long *b, *t;
    cudaMalloc(&b, 8); cudaMalloc(&t, 8);
    for (int bins : {1, 2, 4, 16, 64, 256}) {
        cudaMemset(b, 0, 8); cudaMemset(t, 0, 8);
        probe<<<148 * 4, 256>>>(2000, b, t, bins);
        unsigned long long hb, ht;
        cudaMemcpy(&hb, b, 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(&ht, t, 8, cudaMemcpyDeviceToHost);
        printf("bins %3d: %llu out-of-lane-order ranks in %llu\n", bins, hb, ht);
    }
    return 0;
}
