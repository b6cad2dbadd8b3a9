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

void dist_sweep(DistGroup& grp, Status* const* st);
// op: 0 sum, 1 min, 2 max (no-op without NCCL)
void dist_allreduce(DistGroup& grp, double* buf, size_t count, int op, cudaStream_t s);
void dist_allreduce_int_min(DistGroup& grp, int* buf, cudaStream_t s);
void dist_allreduce_int_sum(DistGroup& grp, int* buf, cudaStream_t s);

bool nccl_available(std::string* why);
void nccl_unique_id(void* out128);
void* nccl_comm_init(const void* id128, int nranks, int rank);
void nccl_comm_destroy(void* comm);

}  // namespace sfm
