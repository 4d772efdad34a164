// pipe.cu -- pipelined executor of host-buffer jobs (agcn_pipe_*, include/agcn.h).
//
// A job is what agcn_propagate_host does: copy the CSR and X in, build the plan (degree sort
// + Alg. 1/2), run `layers` SpMMs, copy Y out.  On a B200 the
// job is bound by the PCIe link (C5: 3.3 GB in, 2.1 GB out, ~7.5 ms of GPU work), and a PCIe
// link is full duplex.  So the executor runs three streams -- copy-in, compute, copy-out --
// and `depth` device buffer sets used round-robin: job k's inputs go in while job k-1's
// result comes out.
//
// Threads: agcn_pipe_submit enqueues the job's copy-in on the calling thread and hands the
// rest to one worker thread, which builds the plan (the plan reads its bucket counts back,
// i.e. it blocks until the job's inputs are resident), enqueues the SpMMs and the copy-out.
// So the caller can enqueue job k+1's copy-in right behind job k's and the copy engine never
// waits for the host.  Cross-job ordering is by events only:
//   copy-in of job k   waits for the compute of the last job in its slot (reads those inputs)
//   compute of job k   waits for its copy-in, and for the copy-out of the last job in its
//                      slot (it overwrites that job's Y buffers)
//   copy-out of job k  waits for its compute.
// A slot is reused only after the worker has enqueued (recorded the events of) its previous
// job, so every event waited on belongs to the right job.
#include <condition_variable>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

#include "internal.h"

namespace agcn {
namespace {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void ensure(size_t bytes) {
        if (bytes <= cap && p) return;
        release();
        AGCN_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
        cap = bytes;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

struct Slot {
    DevBuf rp, ci, va, x, y0, y1;
    cudaEvent_t in_done = nullptr;       // copy-in of the slot's last job complete
    cudaEvent_t compute_done = nullptr;  // its SpMMs complete (inputs free)
    cudaEvent_t out_done = nullptr;      // its copy-out complete (Y buffers free)
    int64_t last_job = -1;               // the slot's last submitted job
    int64_t enqueued_job = -1;           // the last of its jobs the worker has fully enqueued
};

struct Job {
    int64_t id;
    int slot;
    const int32_t* rowptr_h;
    int64_t n, nnz, n_cols;
    int32_t F, layers, base;
    float* Y_h;
};

struct DeviceScope {  // run on the executor's device, restore the caller's
    int prev = -1;
    explicit DeviceScope(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) AGCN_CUDA(cudaSetDevice(dev));
    }
    ~DeviceScope() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace
}  // namespace agcn

struct agcn_pipe_s {
    int device = 0;
    agcn_opts_t opts{};
    cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
    std::vector<agcn::Slot> slots;
    int64_t next = 0;

    std::thread worker;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<agcn::Job> queue;
    bool stop = false;
    int64_t finished = 0;                 // jobs the worker has fully enqueued (or failed)
    agcn_status_t err = AGCN_OK;          // first error of an asynchronous part, until wait
    std::string err_msg;

    void run();
    void process(const agcn::Job& j);
    void release() {
        for (auto& sl : slots) {
            for (agcn::DevBuf* b : {&sl.rp, &sl.ci, &sl.va, &sl.x, &sl.y0, &sl.y1}) b->release();
            for (cudaEvent_t e : {sl.in_done, sl.compute_done, sl.out_done})
                if (e) cudaEventDestroy(e);
        }
        slots.clear();
        for (cudaStream_t s : {s_in, s_comp, s_out})
            if (s) cudaStreamDestroy(s);
        s_in = s_comp = s_out = nullptr;
    }
};

// The worker's part of job j: plan, SpMMs, copy-out.  Whatever happens, the slot's events are
// re-recorded after this job's work so that the next job in the slot orders after it.
void agcn_pipe_s::process(const agcn::Job& j) {
    using namespace agcn;
    Slot& sl = slots[j.slot];
    struct Tail {
        Slot& sl;
        agcn_pipe_s* p;
        ~Tail() {
            cudaEventRecord(sl.compute_done, p->s_comp);
            cudaStreamWaitEvent(p->s_out, sl.compute_done, 0);
            cudaEventRecord(sl.out_done, p->s_out);
        }
    };
    struct PlanGuard {
        agcn_plan_s* p = nullptr;
        ~PlanGuard() {
            if (p) {
                free_plan_arrays(p);  // stream-ordered on the compute stream
                delete p;
            }
        }
    } pg;
    Tail tail{sl, this};
    AGCN_CUDA(cudaStreamWaitEvent(s_comp, sl.in_done, 0));
    agcn_opts_t o = opts;
    o.stream = s_comp;
    auto* rp = static_cast<int32_t*>(sl.rp.p);
    auto* ci = static_cast<int32_t*>(sl.ci.p);
    auto* va = static_cast<float*>(sl.va.p);
    pg.p = build_plan(rp, ci - j.base, j.n, j.nnz, o);
    agcn_spmm_opts_t so;
    agcn_default_spmm_opts(&so);
    const float* cur = static_cast<float*>(sl.x.p);
    float* ybuf[2] = {static_cast<float*>(sl.y0.p), static_cast<float*>(sl.y1.p)};
    for (int l = 0; l < j.layers; ++l) {
        float* out = ybuf[l & 1];
        spmm_launch(pg.p, va - j.base, cur, j.F, out, s_comp, so);
        cur = out;
    }
    AGCN_CUDA(cudaEventRecord(sl.compute_done, s_comp));
    AGCN_CUDA(cudaStreamWaitEvent(s_out, sl.compute_done, 0));
    AGCN_CUDA(cudaMemcpyAsync(j.Y_h, cur, sizeof(float) * (size_t)j.n * j.F, cudaMemcpyDeviceToHost, s_out));
}

void agcn_pipe_s::run() {
    cudaSetDevice(device);
    for (;;) {
        agcn::Job j;
        {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return stop || !queue.empty(); });
            if (queue.empty()) return;  // stop requested and nothing left
            j = queue.front();
        }
        const agcn_status_t st = agcn::guarded([&] { process(j); });
        std::string msg = st != AGCN_OK ? std::string(agcn::last_message()) : std::string();
        {
            std::lock_guard<std::mutex> lk(mu);
            queue.pop_front();
            slots[j.slot].enqueued_job = j.id;
            ++finished;
            if (st != AGCN_OK && err == AGCN_OK) {
                err = st;
                err_msg = msg;
            }
        }
        cv.notify_all();
    }
}

namespace {

void sync_all(agcn_pipe_s* p) {
    cudaError_t e = cudaSuccess;
    for (cudaStream_t s : {p->s_in, p->s_comp, p->s_out}) {
        const cudaError_t r = cudaStreamSynchronize(s);
        if (e == cudaSuccess) e = r;
    }
    if (e != cudaSuccess) throw agcn::Error{agcn::cuda_status(e), std::string("agcn_pipe: ") + cudaGetErrorString(e)};
}

// block until the worker has enqueued every submitted job; hand back its first error
void drain(agcn_pipe_s* p) {
    std::unique_lock<std::mutex> lk(p->mu);
    p->cv.wait(lk, [&] { return p->finished == p->next; });
    if (p->err != AGCN_OK) {
        const agcn::Error e{p->err, p->err_msg};
        p->err = AGCN_OK;
        p->err_msg.clear();
        throw e;
    }
}

}  // namespace

extern "C" {

agcn_pipe_t agcn_pipe_create(int32_t depth, const agcn_opts_t* opts) {
    agcn_pipe_s* p = nullptr;
    const agcn_status_t st = agcn::guarded([&] {
        p = new agcn_pipe_s();
        AGCN_CUDA(cudaGetDevice(&p->device));
        if (opts)
            p->opts = *opts;
        else
            agcn_default_opts(&p->opts);
        AGCN_CHECK(p->opts.col_nparts == 0, AGCN_ERR_INVALID_ARG, "padded layouts are not supported here");
        p->opts.stream = nullptr;
        for (cudaStream_t* s : {&p->s_in, &p->s_comp, &p->s_out})
            AGCN_CUDA(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
        p->slots.resize(depth > 0 ? depth : 2);
        for (auto& sl : p->slots)
            for (cudaEvent_t* e : {&sl.in_done, &sl.compute_done, &sl.out_done})
                AGCN_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        p->worker = std::thread([p] { p->run(); });
    });
    if (st != AGCN_OK && p) {
        p->release();
        delete p;
        p = nullptr;
    }
    return p;
}

agcn_status_t agcn_pipe_submit(agcn_pipe_t pipe, const int32_t* rowptr_h, const int32_t* colidx_h,
                               const float* vals_h, int64_t n, int64_t nnz, const float* X_h, int32_t F,
                               int32_t layers, float* Y_h) {
    using namespace agcn;
    return guarded([&] {
        AGCN_CHECK(pipe && rowptr_h && X_h && Y_h && F > 0 && layers >= 1 && n >= 0 && nnz >= 0,
                   AGCN_ERR_INVALID_ARG, "bad argument");
        AGCN_CHECK(nnz == 0 || (colidx_h && vals_h), AGCN_ERR_INVALID_ARG, "colidx / vals is NULL");
        AGCN_CHECK(nnz < (1ll << 31) && n < (1ll << 31) - 1, AGCN_ERR_INVALID_ARG, "n, nnz must be < 2^31");
        const agcn_opts_t& po = pipe->opts;
        const int64_t n_cols = po.n_cols > 0 ? po.n_cols : n;
        AGCN_CHECK(layers == 1 || n_cols == n, AGCN_ERR_INVALID_ARG, "layers > 1 needs a square A");
        AGCN_CHECK((int64_t)rowptr_h[n] - rowptr_h[0] == nnz, AGCN_ERR_BAD_CSR, "rowptr[n] - rowptr[0] != nnz");
        DeviceScope dev(pipe->device);
        const int si = (int)(pipe->next % (int64_t)pipe->slots.size());
        Slot& sl = pipe->slots[si];
        {   // the slot's previous job must be enqueued by the worker (its events recorded)
            std::unique_lock<std::mutex> lk(pipe->mu);
            pipe->cv.wait(lk, [&] { return sl.enqueued_job == sl.last_job; });
        }
        const size_t xb = sizeof(float) * (size_t)n_cols * F, yb = sizeof(float) * (size_t)n * F;
        const size_t rb = sizeof(int32_t) * (size_t)(n + 1), eb = sizeof(int32_t) * (size_t)nnz;
        const bool grow = sl.rp.cap < rb || sl.ci.cap < eb || sl.va.cap < eb || sl.x.cap < xb ||
                          sl.y0.cap < yb || (layers > 1 && sl.y1.cap < yb);
        if (grow && sl.last_job >= 0) AGCN_CUDA(cudaEventSynchronize(sl.out_done));  // slot idle
        sl.rp.ensure(rb);
        sl.ci.ensure(eb);
        sl.va.ensure(eb);
        sl.x.ensure(xb);
        sl.y0.ensure(yb);
        if (layers > 1) sl.y1.ensure(yb);

        // copy-in (colidx_h / vals_h are indexed by rowptr values: copy the [rowptr[0], rowptr[n]) run)
        const int32_t base = rowptr_h[0];
        if (sl.last_job >= 0) AGCN_CUDA(cudaStreamWaitEvent(pipe->s_in, sl.compute_done, 0));
        AGCN_CUDA(cudaMemcpyAsync(sl.rp.p, rowptr_h, rb, cudaMemcpyHostToDevice, pipe->s_in));
        if (nnz) {
            AGCN_CUDA(cudaMemcpyAsync(sl.ci.p, colidx_h + base, eb, cudaMemcpyHostToDevice, pipe->s_in));
            AGCN_CUDA(cudaMemcpyAsync(sl.va.p, vals_h + base, eb, cudaMemcpyHostToDevice, pipe->s_in));
        }
        AGCN_CUDA(cudaMemcpyAsync(sl.x.p, X_h, xb, cudaMemcpyHostToDevice, pipe->s_in));
        // the Y buffers of the slot's previous job must be copied out before this job's compute
        if (sl.last_job >= 0) AGCN_CUDA(cudaStreamWaitEvent(pipe->s_in, sl.out_done, 0));
        AGCN_CUDA(cudaEventRecord(sl.in_done, pipe->s_in));

        Job j{pipe->next, si, rowptr_h, n, nnz, n_cols, F, layers, base, Y_h};
        {
            std::lock_guard<std::mutex> lk(pipe->mu);
            sl.last_job = j.id;
            pipe->queue.push_back(j);
            ++pipe->next;
        }
        pipe->cv.notify_all();
    });
}

agcn_status_t agcn_pipe_wait(agcn_pipe_t pipe) {
    return agcn::guarded([&] {
        AGCN_CHECK(pipe, AGCN_ERR_INVALID_ARG, "NULL pipe");
        agcn::DeviceScope dev(pipe->device);
        // every job's copies finish before this returns, also when one job failed (the caller
        // may read or free the other jobs' Y buffers right after an error)
        try {
            drain(pipe);
        } catch (...) {
            try { sync_all(pipe); } catch (...) {}
            throw;
        }
        sync_all(pipe);
    });
}

agcn_status_t agcn_pipe_destroy(agcn_pipe_t pipe) {
    if (!pipe) return AGCN_OK;
    const agcn_status_t st = agcn_pipe_wait(pipe);
    {
        std::lock_guard<std::mutex> lk(pipe->mu);
        pipe->stop = true;
    }
    pipe->cv.notify_all();
    if (pipe->worker.joinable()) pipe->worker.join();
    agcn::guarded([&] {
        agcn::DeviceScope dev(pipe->device);
        pipe->release();
    });
    delete pipe;
    return st;
}

}  // extern "C"
