// Probe: device-set conditional IF nodes in a CUDA graph, built with stream
// capture into the body graph (design aid for the graph launch path).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_decide(cudaGraphConditionalHandle h, const int* flag) { cudaGraphSetConditional(h, *flag ? 1u : 0u); }
__global__ void k_body(int* counter) { atomicAdd(counter, 1); }
__global__ void k_after(int* counter) { atomicAdd(counter, 100); }

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

int main() {
    int *flag, *counter;
    CK(cudaMalloc(&flag, 4));
    CK(cudaMalloc(&counter, 4));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 0, 0));
    // segment 1: decide (captured into g)
    CK(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    k_decide<<<1, 1, 0, s>>>(h, flag);
    cudaStreamCaptureStatus st;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    CK(cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &ndeps));
    // conditional node after it
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    CK(cudaGraphAddNode(&cn, g, deps, ndeps, &cp));
    CK(cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies));
    k_after<<<1, 1, 0, s>>>(counter);
    CK(cudaStreamEndCapture(s, &g));
    // body: capture into the conditional's body graph
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaStream_t s2;
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    CK(cudaStreamBeginCaptureToGraph(s2, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    k_body<<<4, 32, 0, s2>>>(counter);
    k_body<<<1, 32, 0, s2>>>(counter);
    CK(cudaStreamEndCapture(s2, &body));
    cudaGraphExec_t ge;
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int f = 0; f < 2; ++f) {
        CK(cudaMemset(counter, 0, 4));
        CK(cudaMemcpy(flag, &f, 4, cudaMemcpyHostToDevice));
        CK(cudaGraphLaunch(ge, s));
        CK(cudaStreamSynchronize(s));
        int c = 0;
        CK(cudaMemcpy(&c, counter, 4, cudaMemcpyDeviceToHost));
        printf("flag=%d counter=%d (expect %d)\n", f, c, f ? 100 + 160 : 100);
    }
    // timing: 1000 launches of a graph with the body off
    int z = 0;
    CK(cudaMemcpy(flag, &z, 4, cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int i = 0; i < 1000; ++i) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("graph launch (3 nodes, body skipped): %.2f us each\n", ms);
    return 0;
}
