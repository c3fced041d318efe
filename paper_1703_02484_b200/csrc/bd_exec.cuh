// bd_exec.cuh -- execution policies for the device-resident step drivers.
//
// A step driver (bd_step.cuh) is written ONCE as uniform control flow over
// data-parallel phases:
//
//     for (i = x.tid(); i < n; i += x.nth()) body(i);   // a phase
//     v = R.close(slot);                                 // barrier + reduced value
//
// and instantiated with
//   ExecGrid  -- persistent cooperative kernel, barrier = grid.sync()
//   ExecBlock -- one CTA, barrier = __syncthreads()      (small N)
//   ExecHost  -- one host thread, barrier = no-op         (tests/hostemu only:
//                runs the identical driver logic on the CPU so control flow
//                can be checked without a GPU; never used by the product)
// Every thread executes the same sequence of barriers; decisions are made
// only on values read after a barrier, so all threads take the same branch.
#pragma once

#include "bd_common.cuh"

#if defined(__CUDACC__)
#include <cooperative_groups.h>
#endif

namespace bd {

typedef unsigned long long u64;

// control block at the head of the workspace
struct Ctl {
    u64 red[8];     // reduction ring (see Red)
    u64 status;     // first error code (BD_ERR_*), 0 = ok
    u64 err_i, err_k;
    u64 scratch[5];
    u64 lists[8];   // worklist lengths (restore_delaunay): two rings of 4
    u64 gen;        // worklist dedup generation
    u64 vgen;       // correct_overlaps: generation of the per-particle overlap stamps
    u64 wgen;       // ph_select_and_flip: last LFMIS round stamp
    u64 bsum[4096]; // per-block partial sums (grid scans)
};

#if defined(__CUDACC__)

BD_DEV u64 ld_volatile(const u64* p) { return *(const volatile u64*)p; }

// warp-aggregated atomic add (most lanes contribute 0)
BD_DEV void atomic_add_u64(u64* p, u64 v) {
    if (v) atomicAdd(p, v);
}

// sum over the warp, one atomic per warp (every lane of the warp must call it)
BD_DEV void warp_atomic_add_u64(u64* p, u64 v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(p, v);
}

// list append from possibly divergent code: the lanes that arrive together
// take one atomic per warp and consecutive slots
BD_DEV u64 warp_append(u64* counter) {
    const unsigned mask = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    u64 base = 0;
    if (lane == leader) base = atomicAdd(counter, (u64)__popc(mask));
    base = __shfl_sync(mask, base, leader);
    return base + (u64)__popc(mask & ((1u << lane) - 1u));
}

// max over the warp, one atomic per warp (every lane of the warp must call it)
BD_DEV void warp_atomic_max_u64(u64* p, u64 v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const u64 w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    if ((threadIdx.x & 31) == 0 && v) atomicMax(p, v);
}

template <int NW>
BD_DEV int64_t block_reduce_sum(int64_t v, int64_t* sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    int64_t t = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sh[k];
    return t;
}

// exclusive scan of one value per thread over the block; returns the block total
BD_DEV int64_t block_excl_scan(int64_t v, int64_t& excl, int64_t* sh) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int64_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    __syncthreads();
    if (lane == 31) sh[w] = inc;
    __syncthreads();
    int64_t before = 0, total = 0;
    for (int k = 0; k < nw; ++k) {
        if (k < w) before += sh[k];
        total += sh[k];
    }
    excl = before + inc - v;
    return total;
}

struct ExecGrid {
    Ctl* ctl;
    BD_DEV int64_t tid() const { return (int64_t)blockIdx.x * blockDim.x + threadIdx.x; }
    BD_DEV int64_t nth() const { return (int64_t)gridDim.x * blockDim.x; }
    BD_DEV bool leader() const { return blockIdx.x == 0 && threadIdx.x == 0; }
    BD_DEV void sync() { cooperative_groups::this_grid().sync(); }
    BD_DEV void add(u64* p, u64 v) { atomic_add_u64(p, v); }
    BD_DEV void umax(u64* p, u64 v) { atomicMax(p, v); }
    BD_DEV void umax_all(u64* p, u64 v) { warp_atomic_max_u64(p, v); }  // every thread calls it
    BD_DEV void add_all(u64* p, u64 v) { warp_atomic_add_u64(p, v); }   // every thread calls it
    BD_DEV void umin(u64* p, u64 v) { atomicMin(p, v); }
    BD_DEV u64 cas(u64* p, u64 cmp, u64 v) { return atomicCAS(p, cmp, v); }
    BD_DEV int32_t fetch_add32(int32_t* p, int32_t v) { return atomicAdd(p, v); }
    BD_DEV u64 fetch_add64(u64* p, u64 v) { return atomicAdd(p, v); }
    BD_DEV u64 append(u64* p) { return warp_append(p); }  // list slot, one atomic per warp
    BD_DEV uint32_t exch32(uint32_t* p, uint32_t v) { return atomicExch(p, v); }
#ifndef BD_GRID_LD_BCAST
#define BD_GRID_LD_BCAST 1
#endif
    // a control word read after a barrier (uniform: every thread calls it):
    // one load per CTA, broadcast through shared memory, instead of every
    // warp of the grid loading the same L2 line right after the barrier
    BD_DEV u64 ld(const u64* p) const {
#if BD_GRID_LD_BCAST
        __shared__ u64 bc;
        __syncthreads();  // earlier readers of bc are done
        if (threadIdx.x == 0) bc = ld_volatile(p);
        __syncthreads();
        return bc;
#else
        return ld_volatile(p);
#endif
    }

    // in-place exclusive scan of a[0..n) (int32), a[n] = total; ends with a barrier
    BD_DEV void exclusive_scan(int32_t* a, int64_t n) {
        __shared__ int64_t sh[32];
        const int64_t nb = gridDim.x, b = blockIdx.x;
        const int64_t R = (n + nb - 1) / nb;
        const int64_t lo = b * R < n ? b * R : n, hi = (b + 1) * R < n ? (b + 1) * R : n;
        int64_t part = 0;
        for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) part += a[i];
        part = block_reduce_sum<32>(part, sh);
        if (threadIdx.x == 0) ctl->bsum[b] = (u64)part;
        sync();
        int64_t pre = 0;
        for (int64_t j = threadIdx.x; j < b; j += blockDim.x) pre += (int64_t)ld_volatile(&ctl->bsum[j]);
        pre = block_reduce_sum<32>(pre, sh);
        int64_t carry = pre;
        for (int64_t base = lo; base < hi; base += blockDim.x) {
            int64_t i = base + threadIdx.x;
            int64_t v = i < hi ? a[i] : 0, ex;
            int64_t tot = block_excl_scan(v, ex, sh);
            if (i < hi) a[i] = (int32_t)(carry + ex);
            carry += tot;
            __syncthreads();
        }
        if (b == nb - 1 && threadIdx.x == 0) a[n] = (int32_t)carry;
        sync();
    }
};

struct ExecBlock {
    Ctl* ctl;
    BD_DEV int64_t tid() const { return threadIdx.x; }
    BD_DEV int64_t nth() const { return blockDim.x; }
    BD_DEV bool leader() const { return threadIdx.x == 0; }
    BD_DEV void sync() {
        __threadfence_block();
        __syncthreads();
    }
    BD_DEV void add(u64* p, u64 v) { atomic_add_u64(p, v); }
    BD_DEV void umax(u64* p, u64 v) { atomicMax(p, v); }
    BD_DEV void umax_all(u64* p, u64 v) { warp_atomic_max_u64(p, v); }  // every thread calls it
    BD_DEV void add_all(u64* p, u64 v) { warp_atomic_add_u64(p, v); }   // every thread calls it
    BD_DEV void umin(u64* p, u64 v) { atomicMin(p, v); }
    BD_DEV u64 cas(u64* p, u64 cmp, u64 v) { return atomicCAS(p, cmp, v); }
    BD_DEV int32_t fetch_add32(int32_t* p, int32_t v) { return atomicAdd(p, v); }
    BD_DEV u64 fetch_add64(u64* p, u64 v) { return atomicAdd(p, v); }
    BD_DEV u64 append(u64* p) { return warp_append(p); }  // list slot, one atomic per warp
    BD_DEV uint32_t exch32(uint32_t* p, uint32_t v) { return atomicExch(p, v); }
    BD_DEV u64 ld(const u64* p) const { return ld_volatile(p); }

    BD_DEV void exclusive_scan(int32_t* a, int64_t n) {
        __shared__ int64_t sh[32];
        int64_t carry = 0;
        for (int64_t base = 0; base < n; base += blockDim.x) {
            int64_t i = base + threadIdx.x;
            int64_t v = i < n ? a[i] : 0, ex;
            int64_t tot = block_excl_scan(v, ex, sh);
            if (i < n) a[i] = (int32_t)(carry + ex);
            carry += tot;
            __syncthreads();
        }
        if (threadIdx.x == 0) a[n] = (int32_t)carry;
        sync();
    }
};

#endif  // __CUDACC__

// host emulation (tests only): one "thread" covering every element in order
struct ExecHost {
    Ctl* ctl;
    int64_t tid() const { return 0; }
    int64_t nth() const { return 1; }
    bool leader() const { return true; }
    void sync() {}
    void add(u64* p, u64 v) { *p += v; }
    void umax(u64* p, u64 v) {
        if (v > *p) *p = v;
    }
    void umax_all(u64* p, u64 v) { umax(p, v); }
    void add_all(u64* p, u64 v) { *p += v; }
    void umin(u64* p, u64 v) {
        if (v < *p) *p = v;
    }
    u64 cas(u64* p, u64 cmp, u64 v) {
        u64 old = *p;
        if (old == cmp) *p = v;
        return old;
    }
    int32_t fetch_add32(int32_t* p, int32_t v) {
        int32_t o = *p;
        *p += v;
        return o;
    }
    u64 fetch_add64(u64* p, u64 v) {
        u64 o = *p;
        *p += v;
        return o;
    }
    u64 append(u64* p) { return (*p)++; }
    uint32_t exch32(uint32_t* p, uint32_t v) {
        uint32_t o = *p;
        *p = v;
        return o;
    }
    u64 ld(const u64* p) const { return *p; }
    void exclusive_scan(int32_t* a, int64_t n) {
        int64_t c = 0;
        for (int64_t i = 0; i < n; ++i) {
            int64_t v = a[i];
            a[i] = (int32_t)c;
            c += v;
        }
        a[n] = (int32_t)c;
    }
};

// Reduction ring: reduction k accumulates into red[k & 7]; whoever opens
// reduction k zeroes red[(k+1) & 7] for the next one.  That slot was last
// read right after the barrier of reduction k-7, so no thread can still be
// reading it, and the barrier closing reduction k publishes the zero before
// reduction k+1 accumulates.  All threads open/close in lockstep.
// Contributions (add) accumulate in a per-thread register and reach the
// slot at close() with one atomic per warp -- not one per element, which
// serialises on the single address (a 1M-particle pass: ~0.7 ms).
template <class X>
struct Red {
    X& x;
    unsigned k;
    u64 acc;
    BD_HD explicit Red(X& x_) : x(x_), k(0), acc(0) {}
    BD_HD u64* open() {
        if (x.leader()) x.ctl->red[(k + 1) & 7] = 0;
        acc = 0;
        return &x.ctl->red[k & 7];
    }
    BD_HD void add(u64 v) { acc += v; }
    BD_HD u64 close(u64* s) {
        x.add_all(s, acc);
        acc = 0;
        x.sync();
        u64 v = x.ld(s);
        ++k;
        return v;
    }
};

}  // namespace bd
