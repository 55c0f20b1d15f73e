// Probe of TMA gather4 swizzle placement (diagnostic, not product code):
// loads rows r0..r3 of a 64 x 32 float tensor (value = row * 100 + col) into
// shared memory at a given byte offset with a given swizzle mode and prints
// where each 16-byte chunk landed.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__global__ void probe(const __grid_constant__ CUtensorMap map, uint32_t off, float* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bar;
    float* dst = reinterpret_cast<float*>(sm + off);
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = -1.f;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(512));
        int r0 = 5, r1 = 6, r2 = 7, r3 = 8, col = 0;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(b)
            : "memory");
        asm volatile(
            "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(b)
            : "memory");
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}

int main() {
    float h[64 * 32];
    for (int r = 0; r < 64; ++r)
        for (int c = 0; c < 32; ++c) h[r * 32 + c] = r * 100 + c;
    float *d, *o;
    cudaMalloc(&d, sizeof(h));
    cudaMalloc(&o, 4096 * 4);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    const CUtensorMapSwizzle modes[] = {CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B};
    const char* names[] = {"128B", "128B_ATOM_32B"};
    const uint32_t offs[] = {0, 128, 256, 384, 512, 1152, 2304};
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 20000);
    for (int mi = 0; mi < 2; ++mi) {
        CUtensorMap map;
        cuuint64_t dims[2] = {32, 64};
        cuuint64_t str[1] = {32 * 4};
        cuuint32_t box[2] = {32, 1};
        cuuint32_t es[2] = {1, 1};
        CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, modes[mi], CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("mode %s encode %d\n", names[mi], int(r));
        for (uint32_t off : offs) {
            probe<<<1, 128, 16384>>>(map, off, o);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) { printf(" off %u: %s\n", off, cudaGetErrorString(e)); return 1; }
            float out[4096];
            cudaMemcpy(out, o, sizeof(out), cudaMemcpyDeviceToHost);
            printf(" off %5u:", off);
            for (int row = 0; row < 4; ++row) {  // logical row -> chunk c landed at physical chunk
                printf(" r%d[", row);
                for (int c = 0; c < 8; ++c) {
                    const float want = (5 + row) * 100 + 4 * c;
                    int where = -1;
                    for (int i = 0; i < 4096; i += 4) if (out[i] == want) where = i;
                    printf("%d%s", where < 0 ? -1 : (where * 4 - int(off)) / 16, c < 7 ? "," : "");
                }
                printf("]");
            }
            printf("\n");
        }
    }
    return 0;
}
