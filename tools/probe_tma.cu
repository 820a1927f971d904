// Probe: 3-D TMA tile load (OOB zero fill) into dynamic shared memory, descriptor as a
// __grid_constant__ parameter; variants: destination offset 0 / 1024-aligned, 2 D vs 3 D.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap pmap, const CUtensorMap* gmap, float* out, int c0, int c1, int c2,
                  int align) {
    const CUtensorMap* mp = gmap ? gmap : &pmap;
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char* base = align ? (unsigned char*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023) : raw;
    float* dst = (float*)base;
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bar)), "r"(40 * 38 * 4) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            ::"r"(saddr(dst)), "l"(mp), "r"(c0), "r"(c1), "r"(c2), "r"(saddr(&bar)) : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n}"
                     : "=r"(ok) : "r"(saddr(&bar)) : "memory");
    for (int i = threadIdx.x; i < 40 * 38; i += blockDim.x) out[i] = dst[i];
}

int run(int nx, int ny, int nz, int l2none) {
    std::vector<float> h(nx * ny * nz);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, 40 * 38 * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    CUtensorMap map;
    memset(&map, 0, sizeof(map));
    const cuuint64_t dims[3] = {nx, ny, nz};
    const cuuint64_t strides[2] = {nx * 4, (cuuint64_t)nx * ny * 4};
    const cuuint32_t box[3] = {40, 38, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, l2none ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("dims %d %d %d l2none %d: encode %d (map %p aligned64=%d)\n", nx, ny, nz, l2none, (int)r, (void*)&map, (int)(((uintptr_t)&map) % 64 == 0));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    CUtensorMap* gm;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &map, sizeof(map), cudaMemcpyHostToDevice);
    for (int glob = 1; glob >= 0; --glob)
    for (int align = 0; align < 2; ++align) {
        for (int z : {-3, 2}) {
            k<<<1, 128, 200000>>>(map, glob ? gm : nullptr, o, -3, -3, z, align);
            cudaError_t e = cudaDeviceSynchronize();
            std::vector<float> ho(40 * 38);
            cudaMemcpy(ho.data(), o, ho.size() * 4, cudaMemcpyDeviceToHost);
            // expected at (hy=5, hx=7): x = 4, y = 2, plane z
            float exp = (z >= 0) ? (float)((z * ny + 2) * nx + 4) : 0.0f;
            printf("glob %d align %d z %d: %s value %g expected %g\n", glob, align, z, cudaGetErrorString(e), ho[5 * 40 + 7], exp);
            if (e != cudaSuccess) return 1;
        }
    }
    cudaFree(d);
    cudaFree(o);
    return 0;
}

int main(int argc, char** argv) {
    int nx = atoi(argv[1]), ny = atoi(argv[2]), nz = atoi(argv[3]), l2 = atoi(argv[4]);
    return run(nx, ny, nz, l2);
}
