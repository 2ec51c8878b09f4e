// Cost of a kernel node in a captured CUDA graph on this GPU: a chain of K
// launches of an (almost) empty kernel, timed with events, for several grid sizes
// and with / without a dependent global load at entry.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o node_probe node_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(const int* flag, int* out) {
    if (flag && *flag) out[blockIdx.x] = 1;
}

int main() {
    int* d;
    cudaMalloc(&d, 1 << 20);
    cudaMemset(d, 0, 1 << 20);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int K = 50;
    int grids[] = {1, 148, 1184, 2368};
    for (int load = 0; load < 2; load++)
        for (int g : grids) {
            cudaGraph_t graph;
            cudaGraphExec_t exec;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int i = 0; i < K; i++) k_empty<<<g, 256, 0, s>>>(load ? d : nullptr, d + 1024);
            cudaStreamEndCapture(s, &graph);
            cudaGraphInstantiate(&exec, graph, 0);
            for (int w = 0; w < 5; w++) cudaGraphLaunch(exec, s);
            cudaStreamSynchronize(s);
            const int R = 50;
            cudaEventRecord(a, s);
            for (int r = 0; r < R; r++) cudaGraphLaunch(exec, s);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("grid %5d load %d: %.2f us per node\n", g, load, 1000.0 * ms / (R * K));
            cudaGraphExecDestroy(exec);
            cudaGraphDestroy(graph);
        }
    return 0;
}
