// launch_floor.cu -- the per-call floor of a chain of dependent kernels in one CUDA graph on this
// B200: K launches of a trivial kernel (griddepcontrol.wait, one load + store of the previous
// launch's output, launch_dependents), with and without programmatic dependent launch, for grids
// of 16 / 48 / 148 CTAs.  Compares with the 2^4 coarse apply's per-call time.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/launch_floor launch_floor.cu && /tmp/launch_floor
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step(const float *in, float *out)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    out[i] = in[i] * 1.0001f + 1.0f;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

static float run(int grid, int K, bool pdl)
{
    float *a, *b;
    cudaMalloc(&a, grid * 128 * sizeof(float));
    cudaMalloc(&b, grid * 128 * sizeof(float));
    cudaMemset(a, 0, grid * 128 * sizeof(float));
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int k = 0; k < K; k++) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(128);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        const float *in = (k & 1) ? b : a;
        float *out = (k & 1) ? a : b;
        void *args[] = {&in, &out};
        cudaLaunchKernelExC(&cfg, (const void *)step, args);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 10; r++) {
        cudaEventRecord(e0, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaFree(a);
    cudaFree(b);
    cudaStreamDestroy(s);
    return best * 1000.f / K;
}

int main()
{
    for (int grid : {16, 48, 148})
        for (int pdl : {0, 1})
            printf("grid %3d  pdl %d : %.3f us per dependent launch\n", grid, pdl, run(grid, 400, pdl));
    return 0;
}
