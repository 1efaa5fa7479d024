// ct_comm.cuh — the exchange steps of the multi-rank path behind one interface.
//
//   NcclComm     one process per GPU: an ncclComm_t (NCCL is dlopen'ed at run time, the copy
//                torch already loaded), every call enqueued on the caller's stream.
//   VirtualComm  P virtual ranks of ONE process on ONE device, for validating the multi-rank
//                code path (slab padding, reduce-scatter into padded slabs, slab g-update, xi
//                all-reduce, all-gather, z-slab sinogram sums and halos) on a single GPU.
//                Each rank is driven by its own host thread on its own stream.  A collective
//                is a host rendezvous of the P threads; the last one to arrive makes a group
//                stream wait on every rank's stream (events), runs device copies and fixed-order
//                sum kernels there, and makes every rank's stream wait on the result.  No kernel
//                ever waits on another kernel: all ordering is stream / event ordering, so the
//                ranks cannot deadlock the device (B200_PROFILING.md's rule for one-GPU stand-ins).
//
// Sums over ranks are taken in rank order 0..P-1 (deterministic for a given P).
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <memory>
#include <mutex>
#include <vector>

namespace ct {

enum CommDType { COMM_F32 = 0, COMM_F64 = 1, COMM_U8 = 2 };

inline size_t comm_elem_bytes(int dt) { return dt == COMM_F64 ? 8 : dt == COMM_F32 ? 4 : 1; }

struct Comm {
    int rank = 0, nranks = 1;
    virtual ~Comm() {}
    virtual const char* kind() const = 0;
    virtual const char* last_err() const = 0;   // message of the last failed call
    // Every call returns 0 on success, nonzero on failure (then last_err() says why).
    // recv[i] = sum over ranks of send[i], i < n (send may equal recv)
    virtual int allreduce_sum(const void* send, void* recv, size_t n, int dt, cudaStream_t st) = 0;
    // recv[i] = sum over ranks q of send_q[rank * n + i], i < n (fp32)
    virtual int reduce_scatter_sum(const float* send, float* recv, size_t n, cudaStream_t st) = 0;
    // recv[q * n + i] = send_q[i] (fp32; send may be recv + rank * n)
    virtual int all_gather(const float* send, float* recv, size_t n, cudaStream_t st) = 0;
    // neighbour exchange along the rank order: recv_lo <- (rank - 1).send_hi, recv_hi <- (rank + 1).send_lo
    virtual int halo(const void* send_lo, const void* send_hi, void* recv_lo, void* recv_hi, size_t n, int dt,
                     cudaStream_t st) = 0;
    // personalised exchange (fp32): send[q] (scount[q] floats) goes to rank q, recv[q] (rcount[q]
    // floats) comes from rank q; q = rank is a local copy; zero counts are skipped.  Every pair
    // of ranks must agree on the counts (rank q's scount[p] = rank p's rcount[q]).
    virtual int alltoallv(const float* const* send, const size_t* scount, float* const* recv, const size_t* rcount,
                          cudaStream_t st) = 0;
};

template <class T>
__global__ void comm_add_kernel(T* __restrict__ dst, const T* __restrict__ src, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] += src[i];
}

// ---------------------------------------------------------------------------
// Virtual ranks
// ---------------------------------------------------------------------------
struct VirtualGroup {
    enum Op { OP_ALLREDUCE = 1, OP_REDUCE_SCATTER = 2, OP_ALL_GATHER = 3, OP_HALO = 4, OP_ALLTOALLV = 5 };
    struct Slot {
        int op;
        const void* send;
        const void* send2;
        void* recv;
        void* recv2;
        size_t n;
        int dt;
        cudaStream_t st;
        std::vector<const float*> vs;   // OP_ALLTOALLV: per-peer buffers and counts
        std::vector<size_t> vsc;
        std::vector<float*> vr;
        std::vector<size_t> vrc;
    };
    int P = 0, device = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long gen = 0;
    int result = 0;
    char err[256] = "";
    std::vector<Slot> slots;
    std::vector<cudaEvent_t> ev_in;
    cudaEvent_t ev_done = nullptr;
    cudaStream_t gst = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    unsigned long long kernels = 0;   // sum / copy work launched (diagnostic)

    int init(int P_, int dev) {
        P = P_;
        device = dev;
        slots.resize(P);
        ev_in.resize(P, nullptr);
        cudaError_t e = cudaStreamCreateWithFlags(&gst, cudaStreamNonBlocking);
        for (int q = 0; q < P && e == cudaSuccess; q++) e = cudaEventCreateWithFlags(&ev_in[q], cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming);
        return e == cudaSuccess ? 0 : -1;
    }
    ~VirtualGroup() {
        for (auto e : ev_in)
            if (e) cudaEventDestroy(e);
        if (ev_done) cudaEventDestroy(ev_done);
        if (gst) cudaStreamDestroy(gst);
        if (tmp) cudaFree(tmp);
    }

    template <class T>
    cudaError_t add(T* dst, const T* src, size_t n) {
        if (n == 0) return cudaSuccess;
        comm_add_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, gst>>>(dst, src, n);
        kernels++;
        return cudaGetLastError();
    }

    // dst = sum_q src_q[off .. off + n) in rank order, through tmp (dst may alias a source)
    cudaError_t sum_into(void* dst, size_t off, size_t n, int dt) {
        const size_t eb = comm_elem_bytes(dt);
        if (n == 0) return cudaSuccess;
        if (tmp_bytes < n * eb) {
            if (tmp) cudaFree(tmp);
            tmp = nullptr;
            tmp_bytes = 0;
            cudaError_t e = cudaMalloc(&tmp, n * eb);
            if (e != cudaSuccess) return e;
            tmp_bytes = n * eb;
        }
        cudaError_t e = cudaMemcpyAsync(tmp, (const char*)slots[0].send + off * eb, n * eb, cudaMemcpyDeviceToDevice, gst);
        for (int q = 1; q < P && e == cudaSuccess; q++) {
            const void* s = (const char*)slots[q].send + off * eb;
            e = dt == COMM_F64 ? add<double>((double*)tmp, (const double*)s, n) : add<float>((float*)tmp, (const float*)s, n);
        }
        if (e == cudaSuccess) e = cudaMemcpyAsync(dst, tmp, n * eb, cudaMemcpyDeviceToDevice, gst);
        return e;
    }

    cudaError_t execute() {
        const Slot& s0 = slots[0];
        for (int q = 1; q < P; q++)
            if (slots[q].op != s0.op || slots[q].n != s0.n || slots[q].dt != s0.dt) {
                snprintf(err, sizeof(err), "virtual ranks: mismatched collectives (rank 0 op %d n %zu, rank %d op %d n %zu)",
                         s0.op, s0.n, q, slots[q].op, slots[q].n);
                return cudaErrorInvalidValue;
            }
        const size_t n = s0.n, eb = comm_elem_bytes(s0.dt);
        cudaError_t e = cudaSuccess;
        for (int q = 0; q < P && e == cudaSuccess; q++) e = cudaStreamWaitEvent(gst, ev_in[q], 0);
        if (e != cudaSuccess) return e;
        switch (s0.op) {
            case OP_ALLREDUCE:
                // sum into rank 0's recv, then broadcast (sources are read before any recv is written:
                // sum_into stages the sum in tmp)
                e = sum_into(slots[0].recv, 0, n, s0.dt);
                for (int q = 1; q < P && e == cudaSuccess; q++)
                    e = cudaMemcpyAsync(slots[q].recv, tmp, n * eb, cudaMemcpyDeviceToDevice, gst);
                break;
            case OP_REDUCE_SCATTER:
                for (int p = 0; p < P && e == cudaSuccess; p++) e = sum_into(slots[p].recv, (size_t)p * n, n, COMM_F32);
                break;
            case OP_ALL_GATHER:
                for (int p = 0; p < P && e == cudaSuccess; p++)
                    for (int q = 0; q < P && e == cudaSuccess; q++) {
                        float* dst = (float*)slots[p].recv + (size_t)q * n;
                        if (dst != slots[q].send)
                            e = cudaMemcpyAsync(dst, slots[q].send, n * 4, cudaMemcpyDeviceToDevice, gst);
                    }
                break;
            case OP_ALLTOALLV:
                for (int p = 0; p < P && e == cudaSuccess; p++)
                    for (int q = 0; q < P && e == cudaSuccess; q++) {
                        // rank q's block for p -> rank p's block from q
                        const size_t c = slots[q].vsc[p];
                        if (c != slots[p].vrc[q]) {
                            snprintf(err, sizeof(err), "virtual ranks: alltoallv count mismatch %d->%d (%zu vs %zu)",
                                     q, p, c, slots[p].vrc[q]);
                            return cudaErrorInvalidValue;
                        }
                        if (c) e = cudaMemcpyAsync(slots[p].vr[q], slots[q].vs[p], c * 4, cudaMemcpyDeviceToDevice, gst);
                    }
                break;
            case OP_HALO:
                for (int p = 0; p < P && e == cudaSuccess; p++) {
                    if (p > 0 && slots[p].recv)
                        e = cudaMemcpyAsync(slots[p].recv, slots[p - 1].send2, n * eb, cudaMemcpyDeviceToDevice, gst);
                    if (e == cudaSuccess && p < P - 1 && slots[p].recv2)
                        e = cudaMemcpyAsync(slots[p].recv2, slots[p + 1].send, n * eb, cudaMemcpyDeviceToDevice, gst);
                }
                break;
            default:
                e = cudaErrorInvalidValue;
        }
        if (e == cudaSuccess) e = cudaEventRecord(ev_done, gst);
        for (int q = 0; q < P && e == cudaSuccess; q++) e = cudaStreamWaitEvent(slots[q].st, ev_done, 0);
        return e;
    }

    // Called by rank `r`'s thread: returns after the collective is enqueued for every rank.
    int collective(int r, const Slot& s, char* errbuf, size_t errlen) {
        cudaError_t e = cudaEventRecord(ev_in[r], s.st);
        std::unique_lock<std::mutex> lk(mu);
        slots[r] = s;
        if (e != cudaSuccess) {
            // still rendezvous (the other ranks would block), but report the failure
            result = -1;
            snprintf(err, sizeof(err), "virtual ranks: cudaEventRecord: %s", cudaGetErrorString(e));
        }
        const unsigned long long my = gen;
        if (++arrived == P) {
            if (result == 0) {
                int dev0 = -1;
                cudaGetDevice(&dev0);
                if (dev0 != device) cudaSetDevice(device);
                cudaError_t x = execute();
                if (dev0 != device && dev0 >= 0) cudaSetDevice(dev0);
                if (x != cudaSuccess) {
                    result = -1;
                    if (!err[0]) snprintf(err, sizeof(err), "virtual ranks: %s", cudaGetErrorString(x));
                }
            }
            arrived = 0;
            gen++;
            lk.unlock();
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != my; });
            lk.unlock();
        }
        if (result != 0) {
            snprintf(errbuf, errlen, "%s", err);
            return -1;
        }
        return 0;
    }
};

struct VirtualComm : Comm {
    std::shared_ptr<VirtualGroup> grp;
    char err[256] = "";
    const char* kind() const override { return "virtual"; }
    const char* last_err() const override { return err; }
    int run(int op, const void* send, const void* send2, void* recv, void* recv2, size_t n, int dt, cudaStream_t st) {
        VirtualGroup::Slot s{};
        s.op = op;
        s.send = send;
        s.send2 = send2;
        s.recv = recv;
        s.recv2 = recv2;
        s.n = n;
        s.dt = dt;
        s.st = st;
        return grp->collective(rank, s, err, sizeof(err));
    }
    int allreduce_sum(const void* send, void* recv, size_t n, int dt, cudaStream_t st) override {
        return run(VirtualGroup::OP_ALLREDUCE, send, nullptr, recv, nullptr, n, dt, st);
    }
    int reduce_scatter_sum(const float* send, float* recv, size_t n, cudaStream_t st) override {
        return run(VirtualGroup::OP_REDUCE_SCATTER, send, nullptr, recv, nullptr, n, COMM_F32, st);
    }
    int all_gather(const float* send, float* recv, size_t n, cudaStream_t st) override {
        return run(VirtualGroup::OP_ALL_GATHER, send, nullptr, recv, nullptr, n, COMM_F32, st);
    }
    int halo(const void* send_lo, const void* send_hi, void* recv_lo, void* recv_hi, size_t n, int dt,
             cudaStream_t st) override {
        return run(VirtualGroup::OP_HALO, send_lo, send_hi, rank > 0 ? recv_lo : nullptr,
                   rank < nranks - 1 ? recv_hi : nullptr, n, dt, st);
    }
    int alltoallv(const float* const* send, const size_t* scount, float* const* recv, const size_t* rcount,
                  cudaStream_t st) override {
        VirtualGroup::Slot s{};
        s.op = VirtualGroup::OP_ALLTOALLV;
        s.dt = COMM_F32;
        s.st = st;
        s.vs.assign(send, send + nranks);
        s.vsc.assign(scount, scount + nranks);
        s.vr.assign(recv, recv + nranks);
        s.vrc.assign(rcount, rcount + nranks);
        return grp->collective(rank, s, err, sizeof(err));
    }
};

}  // namespace ct
