#include <cuda_runtime.h>
#include <cstdio>
__global__ void k_body(int* ctr, cudaGraphConditionalHandle h) {
    int c = atomicAdd(ctr, 1) + 1;
    cudaGraphSetConditional(h, c < 10 ? 1 : 0);
}
int main() {
    int* ctr; cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
    printf("add %d\n", e);
    cudaGraph_t body = p.conditional.phGraph_out[0];
    cudaStream_t s; cudaStreamCreate(&s);
    e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    printf("cap %d\n", e);
    k_body<<<1,1,0,s>>>(ctr, h);
    cudaGraph_t out; e = cudaStreamEndCapture(s, &out); printf("end %d\n", e);
    cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0); printf("inst %d\n", e);
    e = cudaGraphLaunch(ex, s); cudaStreamSynchronize(s);
    int hc; cudaMemcpy(&hc, ctr, 4, cudaMemcpyDeviceToHost); printf("ctr %d err %d\n", hc, cudaGetLastError());
}
