// graph.cu -- agcn_graph_*: `layers` SpMMs captured once in a CUDA graph (include/agcn.h).
//
// Small graphs (C1, C2) are bound by kernel-launch latency, not by the GPU: a layer is ~5 us of
// kernel behind ~15 us of host launch path.  The graph replaces the per-layer host path by one
// cudaGraphLaunch.  Capture runs on a private stream after one eager warm-up pass (which grows
// the plan's scratch: no allocation happens inside the capture) and after the plan is complete
// on its own stream, so the captured SpMMs need no cross-stream event (plan->capturing).
#include "internal.h"

struct agcn_graph_s {
    cudaStream_t s = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int device = 0;
    agcn_plan_s* plan = nullptr;  // counted in plan->n_graphs while the graph lives
};

extern "C" {

agcn_graph_t agcn_graph_create(agcn_plan_t plan, const float* vals, const float* X, int32_t F, int32_t layers,
                               float* ybuf0, float* ybuf1) {
    using namespace agcn;
    agcn_graph_s* g = nullptr;
    const agcn_status_t st = guarded([&] {
        AGCN_CHECK(plan && X && ybuf0 && F > 0 && layers >= 1, AGCN_ERR_INVALID_ARG, "bad argument");
        AGCN_CHECK(layers == 1 || ybuf1, AGCN_ERR_INVALID_ARG, "layers > 1 needs ybuf1");
        AGCN_CHECK(layers == 1 || plan->n_cols == plan->n, AGCN_ERR_INVALID_ARG, "layers > 1 needs a square A");
        AGCN_CHECK(plan->nnz == 0 || vals, AGCN_ERR_INVALID_ARG, "vals is NULL");
        g = new agcn_graph_s();
        AGCN_CUDA(cudaGetDevice(&g->device));
        AGCN_CUDA(cudaStreamCreateWithFlags(&g->s, cudaStreamNonBlocking));
        agcn_spmm_opts_t so;
        agcn_default_spmm_opts(&so);
        float* yb[2] = {ybuf0, ybuf1};
        auto run = [&] {
            const float* cur = X;
            for (int l = 0; l < layers; ++l) {
                spmm_launch(plan, vals, cur, F, yb[l & 1], g->s, so);
                cur = yb[l & 1];
            }
        };
        run();                                   // warm-up: plan complete, scratch grown
        AGCN_CUDA(cudaStreamSynchronize(g->s));
        plan->capturing = true;
        struct Off {
            agcn_plan_s* p;
            ~Off() { p->capturing = false; }
        } off{plan};
        AGCN_CUDA(cudaStreamBeginCapture(g->s, cudaStreamCaptureModeThreadLocal));
        try {
            run();
        } catch (...) {
            cudaGraph_t dead = nullptr;
            cudaStreamEndCapture(g->s, &dead);
            if (dead) cudaGraphDestroy(dead);
            throw;
        }
        AGCN_CUDA(cudaStreamEndCapture(g->s, &g->graph));
        AGCN_CUDA(cudaGraphInstantiate(&g->exec, g->graph, 0));
        g->plan = plan;
        plan->n_graphs.fetch_add(1);
    });
    if (st != AGCN_OK && g) {
        if (g->exec) cudaGraphExecDestroy(g->exec);
        if (g->graph) cudaGraphDestroy(g->graph);
        if (g->s) cudaStreamDestroy(g->s);
        delete g;
        g = nullptr;
    }
    return g;
}

agcn_status_t agcn_graph_launch(agcn_graph_t g, agcn_stream_t stream) {
    return agcn::guarded([&] {
        AGCN_CHECK(g && g->exec, AGCN_ERR_INVALID_ARG, "NULL graph");
        cudaStream_t s = (cudaStream_t)stream;
        agcn_plan_s* p = g->plan;
        AGCN_CUDA(cudaGraphLaunch(g->exec, s));
        agcn::count_launch();
        // order agcn_plan_destroy (stream-ordered on the plan's stream) after this replay
        if (s != p->stream) {
            if (!p->last_use) AGCN_CUDA(cudaEventCreateWithFlags(&p->last_use, cudaEventDisableTiming));
            AGCN_CUDA(cudaEventRecord(p->last_use, s));
        }
    });
}

agcn_status_t agcn_graph_destroy(agcn_graph_t g) {
    return agcn::guarded([&] {
        if (!g) return;
        if (g->plan) g->plan->n_graphs.fetch_sub(1);
        if (g->exec) cudaGraphExecDestroy(g->exec);
        if (g->graph) cudaGraphDestroy(g->graph);
        if (g->s) cudaStreamDestroy(g->s);
        delete g;
    });
}

}  // extern "C"
