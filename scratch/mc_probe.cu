// Probe: which cuMulticastCreate parameters does this B200 accept?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
int main() {
    cudaFree(0);
    CUdevice dev; cuDeviceGet(&dev, 0);
    int sup = 0; cuDeviceGetAttribute(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    printf("multicast supported %d\n", sup);
    for (unsigned nd : {1u, 2u}) for (unsigned long long ht : {0ull, (unsigned long long)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, (unsigned long long)CU_MEM_HANDLE_TYPE_FABRIC}) {
        CUmulticastObjectProp p{}; p.numDevices = nd; p.handleTypes = ht; p.size = 2 << 20;
        size_t g = 0; CUresult rg = cuMulticastGetGranularity(&g, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
        p.size = g ? ((p.size + g - 1) / g) * g : p.size;
        CUmemGenericAllocationHandle h; CUresult r = cuMulticastCreate(&h, &p);
        const char* s = nullptr; cuGetErrorString(r, &s);
        printf("numDevices %u handleTypes %llu: gran rc %d g %zu, create rc %d (%s)\n", nd, ht, (int)rg, g, (int)r, s);
        if (r == CUDA_SUCCESS) {
            CUresult ra = cuMulticastAddDevice(h, dev); cuGetErrorString(ra, &s); printf("   add device rc %d (%s)\n", (int)ra, s);
            cuMemRelease(h);
        }
    }
    return 0;
}
