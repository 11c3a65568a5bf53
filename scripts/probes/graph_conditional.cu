#include <cuda_runtime.h>
#include <cstdio>
__global__ void setc(cudaGraphConditionalHandle h, int* ctr, int lim) {
    int v = ++(*ctr);
    cudaGraphSetConditional(h, v < lim ? 1u : 0u);
}
int main() {
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    cudaGraphNode_t n; cudaGraphAddNode(&n, g, nullptr, 0, &p);
    cudaGraph_t body = p.conditional.phGraph_out[0];
    int* ctr; cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
    int lim = 10;
    void* args[] = {&h, &ctr, &lim};
    cudaKernelNodeParams kp = {}; kp.func = (void*)setc; kp.gridDim = dim3(1); kp.blockDim = dim3(1); kp.kernelParams = args;
    cudaGraphNode_t kn; cudaGraphAddKernelNode(&kn, body, nullptr, 0, &kp);
    cudaGraphExec_t ex; cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
    printf("inst %s\n", cudaGetErrorString(e));
    e = cudaGraphLaunch(ex, 0); cudaDeviceSynchronize();
    int v; cudaMemcpy(&v, ctr, 4, cudaMemcpyDeviceToHost);
    printf("launch %s ctr=%d\n", cudaGetErrorString(e), v);
}
