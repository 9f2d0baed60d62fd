// Host cost of the enqueue primitives the eager path uses: cuTensorMapEncodeTiled, cudaLaunchKernelEx
// (plain / PDL attribute / cluster attribute), cudaEventRecord + cudaStreamWaitEvent, cudaGraphLaunch.
// nvcc -O2 -gencode arch=compute_100a,code=sm_100a launch_cost.cu -lcuda -o /tmp/launch_cost
#include <chrono>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

__global__ void empty_kernel(CUtensorMap m, int x) {
    if (x == 12345) printf("%p\n", &m);
}

template <class F>
double per_call_us(int n, F &&f) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f(i);
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / n;
}

int main() {
    cudaFree(0);
    void *buf;
    cudaMalloc(&buf, 64 << 20);
    cudaStream_t st, st2;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&st2, cudaStreamNonBlocking);
    CUtensorMap m;
    cuuint64_t dims[4] = {64, 32, 32, 128};
    cuuint64_t strides[3] = {128, 128 * 32, 128 * 32 * 32};
    cuuint32_t box[4] = {64, 32, 1, 6}, es[4] = {1, 1, 1, 1};
    const int N = 20000;
    double enc = per_call_us(N, [&](int i) {
        dims[3] = 128 + (i & 7);
        cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    });
    auto launch = [&](int attrs_kind) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(148);
        cfg.blockDim = dim3(640);
        cfg.dynamicSmemBytes = 0;
        cfg.stream = st;
        cudaLaunchAttribute at[2];
        int na = 0;
        if (attrs_kind & 1) {
            at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[na++].val.programmaticStreamSerializationAllowed = 1;
        }
        if (attrs_kind & 2) {
            at[na].id = cudaLaunchAttributeClusterDimension;
            at[na].val.clusterDim.x = 2;
            at[na].val.clusterDim.y = 1;
            at[na++].val.clusterDim.z = 1;
        }
        cfg.attrs = at;
        cfg.numAttrs = na;
        double t = 0;
        for (int rep = 0; rep < 10; ++rep) {   // 400 per burst: the launch queue never fills
            t += per_call_us(400, [&](int) { cudaLaunchKernelEx(&cfg, empty_kernel, m, 0); });
            cudaStreamSynchronize(st);
        }
        return t / 10;
    };
    double l0 = launch(0);
    cudaStreamSynchronize(st);
    double l1 = launch(1);
    cudaStreamSynchronize(st);
    double l2 = launch(3);
    cudaStreamSynchronize(st);
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    double evw = per_call_us(N, [&](int) {
        cudaEventRecord(ev, st);
        cudaStreamWaitEvent(st2, ev, 0);
    });
    cudaStreamSynchronize(st);
    cudaStreamSynchronize(st2);
    // a 5-kernel graph
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    for (int k = 0; k < 5; ++k) empty_kernel<<<148, 640, 0, st>>>(m, 0);
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    double gl = 0;
    for (int rep = 0; rep < 10; ++rep) {
        gl += per_call_us(100, [&](int) { cudaGraphLaunch(ge, st); }) / 10;
        cudaStreamSynchronize(st);
    }
    cudaStreamSynchronize(st);
    double q = per_call_us(N, [&](int) { cudaStreamQuery(st); });
    double pk = per_call_us(N, [&](int) { cudaPeekAtLastError(); });
    printf("cuTensorMapEncodeTiled %.3f us\nlaunchEx plain %.3f us\nlaunchEx PDL %.3f us\nlaunchEx PDL+cluster %.3f us\n"
           "eventRecord+streamWait %.3f us\ngraphLaunch (5 kernels) %.3f us\nstreamQuery %.3f us\npeekAtLastError %.3f us\n",
           enc, l0, l1, l2, evw, gl, q, pk);
    return 0;
}
