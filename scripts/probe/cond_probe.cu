// Feasibility probe: a conditional IF node inserted into a stream capture, its body
// captured on a second stream (cudaStreamBeginCaptureToGraph), the predicate set from a kernel.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_pred(cudaGraphConditionalHandle h, const int* flag) { cudaGraphSetConditional(h, *flag ? 1u : 0u); }
__global__ void k_add(int* x, int v) { atomicAdd(x, v); }

int main() {
    cudaStream_t s, b;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    int *flag, *x;
    cudaMalloc(&flag, 4);
    cudaMalloc(&x, 4);
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    k_add<<<1, 1, 0, s>>>(x, 1);
    // conditional node after the current capture frontier
    cudaStreamCaptureStatus st;
    cudaGraph_t cg;
    const cudaGraphNode_t* deps;
    size_t ndeps;
    cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &ndeps);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, cg, 0, 0);
    k_pred<<<1, 1, 0, s>>>(h, flag);
    cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &ndeps);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    cudaError_t e = cudaGraphAddNode(&cn, cg, deps, ndeps, &cp);
    printf("add cond node: %s\n", cudaGetErrorString(e));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(b, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    printf("begin body capture: %s\n", cudaGetErrorString(e));
    k_add<<<1, 1, 0, b>>>(x, 10);
    k_add<<<1, 1, 0, b>>>(x, 100);
    cudaGraph_t bg;
    e = cudaStreamEndCapture(b, &bg);
    printf("end body capture: %s\n", cudaGetErrorString(e));
    e = cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies);
    printf("update deps: %s\n", cudaGetErrorString(e));
    k_add<<<1, 1, 0, s>>>(x, 1000);
    e = cudaStreamEndCapture(s, &g);
    printf("end capture: %s\n", cudaGetErrorString(e));
    cudaGraphExec_t ge;
    e = cudaGraphInstantiate(&ge, g, 0);
    printf("instantiate: %s\n", cudaGetErrorString(e));
    for (int f = 0; f < 2; f++) {
        cudaMemset(x, 0, 4);
        cudaMemcpy(flag, &f, 4, cudaMemcpyHostToDevice);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        int hx;
        cudaMemcpy(&hx, x, 4, cudaMemcpyDeviceToHost);
        printf("flag=%d -> x=%d (expect %d) %s\n", f, hx, f ? 1111 : 1001, cudaGetErrorString(cudaGetLastError()));
    }
    // timing: empty-body skip vs always
    return 0;
}
