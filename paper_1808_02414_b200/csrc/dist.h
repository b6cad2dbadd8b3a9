// Distributed dense sweep state (see dist.cu).
#pragma once

#include "kernels.cuh"

#include <nccl.h>

#include <string>
#include <vector>

namespace sfm {

// One rank's share of the distributed dense stage: its panels' columns, the
// Linv blocks it factors, the panel ring and four streams (critical path,
// trailing update, inverse, communication).
struct RankDense {
    static constexpr int NB = 4;  // ring slots
    Ownership ow{1, 0, 3};
    int Npad = 0, K = 0, ncl = 0;
    long long ld = 0;
    DBuf Z, Linv, piv, ring, range;
    double* zp = nullptr;
    double* linv = nullptr;
    double* pv = nullptr;
    double* ringp = nullptr;
    double* rangep = nullptr;
    cudaStream_t s = nullptr, s2 = nullptr, s3 = nullptr, sc = nullptr;
    cudaEvent_t eL[NB], eB[NB], eRest[NB], eT[NB], eU[NB];
    cudaEvent_t eX2, eX3, eXc, eIn;
    void init(int device);
    void release();
    void setup(const Ownership& o, int Npad, long long ld);
    size_t slot_doubles() const { return (size_t)Npad * ow.G * kNB + (size_t)ow.G * kNB * kNB; }
    double* slot(int p) { return ringp + (size_t)(p % NB) * slot_doubles(); }
};

// The ranks this process drives: all R of them when ranks are emulated on
// one device (nccl == nullptr), else its own one with an NCCL communicator.
struct DistGroup {
    std::vector<RankDense*> ranks;
    void* nccl = nullptr;
};

// Pair blocks grouped by the rank owning their block column (1D panel
// ownership), so one reduce-scatter hands each rank exactly its blocks:
// group g = segments perm[off[g] .. off[g] + cnt[g]), padded to gmax blocks.
struct SegGroups {
    int R = 1, gmax = 1;
    std::vector<int> cnt, off;
    int* perm = nullptr;
    int* d_off = nullptr;
    int* d_cnt = nullptr;
    DBuf buf_owner, buf_owner2, buf_ids, buf_perm, buf_cnt;
    void plan(const ColMap& cm, const Ownership& ow, const unsigned int* ukeys, int nseg, Workspace& ws,
              cudaStream_t s);
    void pack(const double* seg, double* send, cudaStream_t s) const;  // R * gmax * 81 doubles
    void scatter(int g, const double* grp, const ColMap& cm, const Ownership& ow, const unsigned int* ukeys,
                 double* Zl, long long ld, cudaStream_t s) const;
    void release() { buf_owner.release(); buf_owner2.release(); buf_ids.release(); buf_perm.release(); buf_cnt.release(); }
};

void dist_sweep(DistGroup& grp, Status* const* st);
// ncclReduceScatter (sum) of R * count doubles: rank r receives slice r (no-op without NCCL)
void dist_reduce_scatter(DistGroup& grp, const double* send, double* recv, size_t count, cudaStream_t s);
// op: 0 sum, 1 min, 2 max (no-op without NCCL)
void dist_allreduce(DistGroup& grp, double* buf, size_t count, int op, cudaStream_t s);
void dist_allreduce_int_min(DistGroup& grp, int* buf, cudaStream_t s);
// op: 0 sum, 1 min, 2 max
void dist_allreduce_ints(DistGroup& grp, int* buf, size_t count, int op, cudaStream_t s);
void dist_allreduce_u8_max(DistGroup& grp, unsigned char* buf, size_t count, cudaStream_t s);
void dist_allreduce_int_sum(DistGroup& grp, int* buf, cudaStream_t s);

bool nccl_available(std::string* why);
void nccl_unique_id(void* out128);
void* nccl_comm_init(const void* id128, int nranks, int rank);
void nccl_comm_destroy(void* comm);

}  // namespace sfm
