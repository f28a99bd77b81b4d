// Design probe (not product code): the persistent step kernel's attention
// unit run in isolation (one CTA, synthetic q/K/V), %globaltimer stamps via
// teal_step_attn.dbg, to separate its own cost from in-kernel effects.
#include "../../paper_2408_14690_b200/csrc/teal_step.cu"
#include <cstdio>
#include <vector>

using namespace teal::step;
namespace teal {
void set_error(const char*, ...) {}
int check_launch(const char*) { return 0; }
}

__global__ void __launch_bounds__(NT, 2) probe(const __grid_constant__ teal_step_plan P, int reps, int L) {
    for (int r = 0; r < reps; ++r) {
        attn_unit(P, P.attns[0], 0, 0, L);
        __syncthreads();
    }
}

int main() {
    const int H = 32, KVH = 8, hd = 128, max_seq = 2048, G = H / KVH;
    for (int L : {16, 41, 64}) {
        float *q, *ctx, *part;
        uint16_t *kc, *vc;
        int *state, *counters, *dep;
        unsigned *tickets;
        unsigned long long* dbg;
        cudaMalloc(&q, H * hd * 4);
        cudaMalloc(&ctx, H * hd * 4);
        cudaMalloc(&part, 1 << 22);
        cudaMalloc(&kc, (size_t)KVH * max_seq * hd * 2);
        cudaMalloc(&vc, (size_t)KVH * max_seq * hd * 2);
        cudaMemset(kc, 0x3c, (size_t)KVH * max_seq * hd * 2);
        cudaMemset(vc, 0x3c, (size_t)KVH * max_seq * hd * 2);
        cudaMemset(q, 0, H * hd * 4);
        cudaMalloc(&state, 8);
        int hs[2] = {L - 1, L};
        cudaMemcpy(state, hs, 8, cudaMemcpyHostToDevice);
        cudaMalloc(&counters, 1 << 16);
        cudaMemset(counters, 0, 1 << 16);
        cudaMalloc(&dep, 64);
        cudaMemset(dep, 0, 64);
        cudaMalloc(&tickets, 4096);
        cudaMemset(tickets, 0, 4096);
        cudaMalloc(&dbg, 4096);
        cudaMemset(dbg, 0, 4096);
        teal_step_attn a = {};
        a.q = q; a.k_cache = kc; a.v_cache = vc; a.ctx = ctx; a.partials = part; a.tickets = tickets;
        a.max_seq = max_seq; a.H = H; a.KVH = KVH; a.hd = hd; a.kv_dtype = TEAL_BF16; a.chunk = 64; a.nchunks = max_seq / 64;
        a.sig_base = 10; a.dep_base = 0; a.dep_target = dep; a.dbg = dbg;
        teal_step_attn* da;
        cudaMalloc(&da, sizeof(a));
        cudaMemcpy(da, &a, sizeof(a), cudaMemcpyHostToDevice);
        teal_step_plan P = {};
        P.attns = da; P.state = state; P.counters = counters;
        cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
        probe<<<1, NT, sizeof(Smem)>>>(P, 3, L);
        cudaDeviceSynchronize();
        unsigned long long h[6];
        cudaMemcpy(h, dbg, 48, cudaMemcpyDeviceToHost);
        printf("L=%4d (chunk 64, 1 CTA, 3rd rep): stage %.2f us, scores %.2f us, softmax+V+store %.2f us, signal %.2f us  err=%s\n", L,
               (h[2] - h[0]) / 1e3, (h[1] - h[2]) / 1e3, (h[4] - h[1]) / 1e3, (h[5] - h[4]) / 1e3, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
