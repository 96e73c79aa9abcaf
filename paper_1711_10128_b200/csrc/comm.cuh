// Rank-to-rank exchanges of the z-slab partition: NCCL over NVLink/NVSwitch in
// production, or an in-process loopback hub (test infrastructure) that runs several ranks of
// one solve as host threads on ONE GPU: every exchange is a rendezvous of the rank threads,
// the copies are device-to-device cudaMemcpyAsync on the receiving rank's stream ordered by
// CUDA events -- no kernel ever waits on another rank, so ranks sharing a GPU cannot deadlock.
#pragma once
#include <condition_variable>
#include <mutex>
#include <vector>

#include <cuda_runtime.h>
#include <nccl.h>

#include "trplk_kernels.h"

namespace trplk {

struct Xfer {  // one point-to-point transfer of `count` elements of `elsize` bytes
    int peer;
    void* ptr;
    size_t count;
};

class Comm {
public:
    virtual ~Comm() {}
    // recv[r * count .. ] <- send of rank r, for every rank r (fixed rank order)
    virtual bool allgather(const void* send, void* recv, size_t count, size_t elsize, cudaStream_t s) = 0;
    // grouped point-to-point: every send matches the peer's recv of the same count
    virtual bool sendrecv(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, size_t elsize,
                          cudaStream_t s) = 0;
    // buf[i] = sum (op 0) or max (op 1) over ranks; host-synchronous, create time only
    virtual bool allreduce_host(double* v, int count, int op, cudaStream_t s, double* dev_tmp) = 0;
    virtual const char* what() const = 0;
};

class NcclComm : public Comm {
public:
    ncclComm_t comm = nullptr;
    ncclResult_t last = ncclSuccess;
    ~NcclComm() override {
        if (comm) ncclCommDestroy(comm);
    }
    static ncclDataType_t dt(size_t elsize) { return elsize == 8 ? ncclInt64 : ncclInt32; }
    bool allgather(const void* send, void* recv, size_t count, size_t elsize, cudaStream_t s) override {
        last = ncclAllGather(send, recv, count * (elsize / 4), ncclInt32, comm, s);
        return last == ncclSuccess;
    }
    bool sendrecv(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, size_t elsize,
                  cudaStream_t s) override {
        if ((last = ncclGroupStart()) != ncclSuccess) return false;
        for (const Xfer& x : recvs)
            if ((last = ncclRecv(x.ptr, x.count * (elsize / 4), ncclInt32, x.peer, comm, s)) != ncclSuccess)
                return false;
        for (const Xfer& x : sends)
            if ((last = ncclSend(x.ptr, x.count * (elsize / 4), ncclInt32, x.peer, comm, s)) != ncclSuccess)
                return false;
        return (last = ncclGroupEnd()) == ncclSuccess;
    }
    bool allreduce_host(double* v, int count, int op, cudaStream_t s, double* tmp) override {
        if (cudaMemcpyAsync(tmp, v, 8 * (size_t)count, cudaMemcpyHostToDevice, s) != cudaSuccess) return false;
        last = ncclAllReduce(tmp, tmp, count, ncclDouble, op == 0 ? ncclSum : ncclMax, comm, s);
        if (last != ncclSuccess) return false;
        if (cudaMemcpyAsync(v, tmp, 8 * (size_t)count, cudaMemcpyDeviceToHost, s) != cudaSuccess) return false;
        return cudaStreamSynchronize(s) == cudaSuccess;
    }
    const char* what() const override { return ncclGetErrorString(last); }
};

// ---------------------------------------------------------------- loopback (one process, one GPU)
struct LoopHub {
    int n;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long phase = 0;
    // posted by each rank for the current exchange
    std::vector<const void*> ag_send;
    std::vector<std::vector<Xfer>> p2p_send;
    std::vector<cudaEvent_t> ready, done;
    explicit LoopHub(int nr) : n(nr), ag_send(nr), p2p_send(nr), ready(nr), done(nr) {
        for (int r = 0; r < n; ++r) {
            cudaEventCreateWithFlags(&ready[r], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming);
        }
    }
    ~LoopHub() {
        for (int r = 0; r < n; ++r) {
            cudaEventDestroy(ready[r]);
            cudaEventDestroy(done[r]);
        }
    }
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const unsigned long long ph = phase;
        if (++arrived == n) {
            arrived = 0;
            ++phase;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return phase != ph; });
        }
    }
};

class LoopComm : public Comm {
public:
    LoopHub* hub;
    int rank;
    cudaError_t last = cudaSuccess;
    LoopComm(LoopHub* h, int r) : hub(h), rank(r) {}
    // post -> barrier -> copy from peers -> record done -> barrier -> wait for peers' done
    bool finish(cudaStream_t s) {
        if ((last = cudaEventRecord(hub->done[rank], s)) != cudaSuccess) return false;
        hub->barrier();
        for (int r = 0; r < hub->n; ++r)
            if (r != rank && (last = cudaStreamWaitEvent(s, hub->done[r], 0)) != cudaSuccess) return false;
        return true;
    }
    bool allgather(const void* send, void* recv, size_t count, size_t elsize, cudaStream_t s) override {
        hub->ag_send[rank] = send;
        if ((last = cudaEventRecord(hub->ready[rank], s)) != cudaSuccess) return false;
        hub->barrier();
        for (int r = 0; r < hub->n; ++r) {
            if (r != rank && (last = cudaStreamWaitEvent(s, hub->ready[r], 0)) != cudaSuccess) return false;
            if ((last = cudaMemcpyAsync((char*)recv + (size_t)r * count * elsize, hub->ag_send[r], count * elsize,
                                        cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
                return false;
        }
        return finish(s);
    }
    bool sendrecv(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, size_t elsize,
                  cudaStream_t s) override {
        hub->p2p_send[rank] = sends;
        if ((last = cudaEventRecord(hub->ready[rank], s)) != cudaSuccess) return false;
        hub->barrier();
        for (const Xfer& rv : recvs) {
            const Xfer* src = nullptr;
            for (const Xfer& sx : hub->p2p_send[rv.peer])
                if (sx.peer == rank) src = &sx;
            if (!src || src->count != rv.count) {
                last = cudaErrorInvalidValue;
                return false;
            }
            if ((last = cudaStreamWaitEvent(s, hub->ready[rv.peer], 0)) != cudaSuccess) return false;
            if (rv.count && (last = cudaMemcpyAsync(rv.ptr, src->ptr, rv.count * elsize, cudaMemcpyDeviceToDevice,
                                                    s)) != cudaSuccess)
                return false;
        }
        return finish(s);
    }
    bool allreduce_host(double* v, int count, int op, cudaStream_t s, double* tmp) override {
        // allgather of the host values through the device, then the same fixed-order reduction
        if ((last = cudaMemcpyAsync(tmp, v, 8 * (size_t)count, cudaMemcpyHostToDevice, s)) != cudaSuccess) return false;
        double* all = tmp + count;
        if (!allgather(tmp, all, (size_t)count, 8, s)) return false;
        std::vector<double> h((size_t)count * hub->n);
        if ((last = cudaMemcpyAsync(h.data(), all, 8 * h.size(), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return false;
        if ((last = cudaStreamSynchronize(s)) != cudaSuccess) return false;
        for (int i = 0; i < count; ++i) {
            double a = h[i];
            for (int r = 1; r < hub->n; ++r) a = op == 0 ? a + h[(size_t)r * count + i] : std::max(a, h[(size_t)r * count + i]);
            v[i] = a;
        }
        return true;
    }
    const char* what() const override { return cudaGetErrorString(last); }
};

// ---------------------------------------------------------------- host callbacks (one GPU, N processes)
// Exchanges staged through host memory and handed to the caller's callbacks (the Python binding
// routes them to a torch.distributed gloo group): device -> host copy, callback, host -> device
// copy, each synchronous on the rank's stream, so no kernel ever waits on another process and
// several processes can share one GPU (tests of the multi-process bootstrap; bench.py --comm host).
class HostComm : public Comm {
public:
    trplk_host_comm cb;
    cudaError_t lastc = cudaSuccess;
    int lastcb = 0;
    std::vector<char> hs, hr;
    explicit HostComm(const trplk_host_comm& c) : cb(c) {}
    bool cu(cudaError_t e) { return (lastc = e) == cudaSuccess; }
    bool allgather(const void* send, void* recv, size_t count, size_t elsize, cudaStream_t s) override {
        const size_t b = count * elsize;
        hs.resize(b);
        if (!cu(cudaMemcpyAsync(hs.data(), send, b, cudaMemcpyDeviceToHost, s)) || !cu(cudaStreamSynchronize(s)))
            return false;
        hr.resize(b * (size_t)nranks);
        if ((lastcb = cb.allgather(hs.data(), hr.data(), b, cb.user)) != 0) return false;
        return cu(cudaMemcpyAsync(recv, hr.data(), hr.size(), cudaMemcpyHostToDevice, s)) && cu(cudaStreamSynchronize(s));
    }
    bool sendrecv(const std::vector<Xfer>& sends, const std::vector<Xfer>& recvs, size_t elsize,
                  cudaStream_t s) override {
        std::vector<std::vector<char>> sb(sends.size()), rb(recvs.size());
        std::vector<int> sp, rp;
        std::vector<const void*> spt;
        std::vector<void*> rpt;
        std::vector<size_t> sn, rn;
        for (size_t i = 0; i < sends.size(); ++i) {
            sb[i].resize(sends[i].count * elsize);
            if (!sb[i].empty() && !cu(cudaMemcpyAsync(sb[i].data(), sends[i].ptr, sb[i].size(), cudaMemcpyDeviceToHost, s)))
                return false;
            sp.push_back(sends[i].peer);
            spt.push_back(sb[i].data());
            sn.push_back(sb[i].size());
        }
        for (size_t i = 0; i < recvs.size(); ++i) {
            rb[i].resize(recvs[i].count * elsize);
            rp.push_back(recvs[i].peer);
            rpt.push_back(rb[i].data());
            rn.push_back(rb[i].size());
        }
        if (!cu(cudaStreamSynchronize(s))) return false;
        if ((lastcb = cb.sendrecv((int)sp.size(), sp.data(), spt.data(), sn.data(), (int)rp.size(), rp.data(),
                                  rpt.data(), rn.data(), cb.user)) != 0)
            return false;
        for (size_t i = 0; i < recvs.size(); ++i)
            if (!rb[i].empty() && !cu(cudaMemcpyAsync(recvs[i].ptr, rb[i].data(), rb[i].size(), cudaMemcpyHostToDevice, s)))
                return false;
        return cu(cudaStreamSynchronize(s));
    }
    bool allreduce_host(double* v, int count, int op, cudaStream_t s, double* tmp) override {
        (void)s;
        (void)tmp;
        return (lastcb = cb.allreduce(v, count, op, cb.user)) == 0;
    }
    const char* what() const override { return lastcb ? "host exchange callback failed" : cudaGetErrorString(lastc); }
    int nranks = 1;
};

}  // namespace trplk
