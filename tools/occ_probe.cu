// Which kernel property limits the tcgen05 tile kernel to one CTA per SM? (development aid)
#include <cstdio>
#include <cstdint>
__global__ void k_plain(int *p) { p[threadIdx.x] = 1; }
__global__ void k_bars(int *p) {
    asm volatile("bar.sync 1, 128;");
    asm volatile("bar.sync 2, 128;");
    asm volatile("bar.sync 3, 128;");
    asm volatile("bar.sync 4, 128;");
    asm volatile("bar.sync 5, 128;");
    p[threadIdx.x] = 1;
}
__global__ void k_tmem(int *p) {
    __shared__ uint32_t base;
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(base));
    p[threadIdx.x] = 1;
}
__global__ void k_mbar(int *p) {
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    __syncthreads();
    p[threadIdx.x] = 1;
}
int main() {
    int occ;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_plain, 128, 0); printf("plain %d\n", occ);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bars, 128, 0); printf("bars %d\n", occ);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tmem, 128, 0); printf("tmem %d\n", occ);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mbar, 128, 0); printf("mbar %d\n", occ);
    return 0;
}
