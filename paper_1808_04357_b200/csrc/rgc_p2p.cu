// rgc_p2p.cu -- RGC_SYNC_P2P: the Allgather of P:303 as one kernel of NVLink stores;
// RGC_SYNC_PULL: no copy at all -- the decompression reads the peers' blocks in place.
//
// rgc_p2p_init maps, with CUDA IPC, every rank's staging area (nranks message
// blocks, slot r = rank r's block) and epoch flags into every other rank.  The
// exchange of epoch e is then a push: k_p2p_push copies the USED part of this
// rank's message (the header's length elements say how much; no
// host round trip as in SIZES_FIRST) into slot `rank` of every rank's staging
// area with posted stores over NVLink/NVSwitch, and its last CTA publishes
// ready[rank] = e in every peer and waits for every peer's ready >= e.  The
// decompression (K6) then reads only local memory.  After K6 a rank publishes
// consumed[rank] = e (k_finish): a pusher overwrites slot `rank` of rank
// q for epoch e+1 only after q's consumed >= e (WAR on the staging slot).
//
// RGC_SYNC_PULL: rgc_p2p_init also maps every peer's message block.  The sync is
// k_pull_publish (ready[rank] = e in every peer); the decompression starts with
// k_pull_wait (every peer's ready >= e) and its kernels (k6_prep, k6_scatter) load the
// peers' pairs straight over NVLink (MsgSrc::tab); then consumed[rank] = e goes to every
// peer, and the producer's next compress waits in K1 (Ws::pull_flags) for every
// consumer's consumed >= e before K2 rewrites the block (WAR on the message block).
//
// Memory model: every pushing CTA fences at system scope before counting itself
// done; the last one fences again and then stores the flags with st.release.sys;
// readers load flags with ld.acquire.sys.  A wait longer than P2PFlags::timeout_ns
// (RGC_P2P_TIMEOUT_S, default 120 s) sets P2PFlags::err and gives up instead of hanging the
// device; the next decompression's k_finish turns it into the context status, which
// rgc_status reports as RGC_ESTATE (the context is then unusable: the epochs are out of step).
//
// k_finish ends every decompression in every sync mode: it ORs the status word (hdr[L],
// RGC_F_NONFINITE) of every rank's block and the timeout mask into the context status, and in
// P2P / PULL mode publishes consumed[rank] = e (replacing a separate "consumed" launch).
#include <cuda_runtime.h>
#include <stdint.h>

#include "rgc_device.cuh"

namespace rgc {

// grid (nb, p): blockIdx.y = destination rank q, nb CTAs share the copy
__global__ void __launch_bounds__(kThreads)
k_p2p_push(const uint8_t *msg, uint8_t *const *stage, P2PFlags *const *peer_flags, P2PFlags *mine,
           int rank, int p, unsigned long long epoch, uint64_t msg_bytes, int L, uint32_t hdr_words,
           uint64_t tab_off, uint64_t tab_bytes) {
    __shared__ uint64_t s_bytes;
    __shared__ int s_last;
    const int q = blockIdx.y, tid = threadIdx.x;
    pdl_wait();   // the compress kernels before it wrote the block (PDL launch)
    if (tid == 0) {
        // used bytes of this rank's block: header + the pairs its length elements count
        const uint32_t *hdr = reinterpret_cast<const uint32_t *>(msg);
        uint64_t words = 0;   // a pair is 2 words, an ASQ index 1 (hdr[L+2+l], include/rgc.h)
        for (int l = 0; l < L; l++) words += (hdr[L + 2 + l] == RGC_MSG_DENSE ? 2ull : 1ull) * hdr[l];
        const uint64_t used = 4ull * hdr_words + 4ull * words;
        s_bytes = used < tab_off ? used : tab_off;
        // rank q reads slot `rank` of its stage until it has decompressed epoch-1
        if (q != rank && epoch > 1) wait_flag(mine, &mine->consumed[q], q, epoch - 1);
    }
    __syncthreads();
    // the used part (header + entries), then the producer's range table at the block's end
    const uint64_t n16 = (s_bytes + 15) / 16, t16 = tab_bytes / 16, toff16 = tab_off / 16;
    const uint4 *src = reinterpret_cast<const uint4 *>(msg);
    uint4 *dst = reinterpret_cast<uint4 *>(stage[q] + (uint64_t)rank * msg_bytes);
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + tid; i < n16 + t16; i += (uint64_t)gridDim.x * kThreads) {
        const uint64_t j = i < n16 ? i : toff16 + (i - n16);
        RGC_DCHECK(j < msg_bytes / 16);
        dst[j] = src[j];
    }
    __threadfence_system();
    __syncthreads();
    if (tid == 0) {
        const unsigned long long total = (unsigned long long)gridDim.x * gridDim.y;
        const unsigned long long old = atomicAdd(&mine->pushed, 1ull);
        s_last = (old + 1 == epoch * total);
    }
    __syncthreads();
    if (!s_last) return;
    // the last CTA: publish "epoch e is in your stage" to every rank, then wait for theirs
    __threadfence_system();
    for (int r = tid; r < p; r += kThreads)
        if (r != rank) st_release_sys(&peer_flags[r]->ready[rank], epoch);
    for (int r = tid; r < p; r += kThreads)
        if (r != rank) wait_flag(mine, &mine->ready[r], r, epoch);
}

// RGC_SYNC_PULL, producer side: this rank's epoch-e message is complete in its own block
// (stream order: the compress kernels finished); publish ready[rank] = e in every peer.
// Nothing is copied -- the consumers' decompression kernels read the block in place.
__global__ void k_pull_publish(P2PFlags *const *peer_flags, int rank, int p,
                               unsigned long long epoch) {
    pdl_wait();   // the compress kernels before it wrote the block
    __threadfence_system();
    for (int q = threadIdx.x; q < p; q += blockDim.x)
        if (q != rank) st_release_sys(&peer_flags[q]->ready[rank], epoch);
}

// RGC_SYNC_PULL, consumer side: wait until every peer's epoch-e block is published; the
// decompression launched behind this kernel reads the peers' blocks over NVLink
__global__ void k_pull_wait(P2PFlags *mine, int rank, int p, unsigned long long epoch) {
    pdl_wait();
    for (int q = threadIdx.x; q < p; q += blockDim.x)
        if (q != rank) wait_flag(mine, &mine->ready[q], q, epoch);
}

// End of a decompression: status of every rank's block -> context status; then (publish)
// consumed[rank] = epoch in every peer.  One block of 64 threads; p <= 64.
__global__ void k_finish(MsgSrc src, int L, int p, P2PFlags *mine, P2PFlags *const *peer_flags,
                         int rank, unsigned long long epoch, int publish, uint32_t *d_stat,
                         volatile uint32_t *h_stat, int need_tab) {
    __shared__ uint32_t s_or;
    pdl_wait();   // the decompression kernels before it are complete (and read the blocks)
    if (threadIdx.x == 0) s_or = 0;
    __syncthreads();
    for (int r = threadIdx.x; r < p; r += blockDim.x) {
        const uint32_t *h = reinterpret_cast<const uint32_t *>(src.of(r));
        uint32_t st = h[L];
        // the decompression read this block's range table: it must have been written
        if (need_tab && h[2 * L + 2] != kTabMarker) st |= kStatNoTable;
        if (st) atomicOr(&s_or, st);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = s_or;
        const unsigned long long tmo = mine ? *(volatile unsigned long long *)&mine->err : 0ull;
        if (tmo) s |= kStatTimeout;
        if (s) {
            const uint32_t before = atomicOr(&d_stat[0], s);
            if (tmo) {   // which peers a wait gave up on (bit q), ranks 0-31 / 32-63
                atomicOr(&d_stat[1], (uint32_t)tmo);
                atomicOr(&d_stat[2], (uint32_t)(tmo >> 32));
            }
            if ((before | s) != before || tmo) {   // mirror into host-mapped memory on change
                h_stat[1] = d_stat[1];
                h_stat[2] = d_stat[2];
                __threadfence_system();
                h_stat[0] = before | s;
                __threadfence_system();
            }
        }
    }
    if (!publish) return;
    __syncthreads();   // every block above was read before a peer may reuse it
    for (int q = threadIdx.x; q < p; q += blockDim.x) {
        if (q == rank) continue;
        __threadfence_system();
        st_release_sys(&peer_flags[q]->consumed[rank], epoch);
    }
}

// rgc_finalize: every peer is done with this rank's memory once it published consumed >= epoch
__global__ void k_wait_consumed(P2PFlags *mine, int rank, int p, unsigned long long epoch,
                                unsigned long long limit_ns) {
    for (int q = threadIdx.x; q < p; q += blockDim.x) {
        if (q == rank) continue;
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_sys(&mine->consumed[q]) < epoch) {
            if (globaltimer_ns() - t0 > limit_ns) { atomicOr(&mine->err, 1ull << (q & 63)); break; }
            __nanosleep(256);
        }
    }
}

cudaError_t launch_finish(const MsgSrc &src, int L, int p, P2PFlags *mine,
                          P2PFlags *const *peer_flags, int rank, unsigned long long epoch,
                          int publish, uint32_t *d_stat, volatile uint32_t *h_stat, cudaStream_t s,
                          int need_tab) {
    return launch_pdl(k_finish, dim3(1), dim3(64), 0, s, src, L, p, mine, peer_flags, rank, epoch,
                      publish, d_stat, h_stat, need_tab);
}

cudaError_t launch_wait_consumed(P2PFlags *mine, int rank, int p, unsigned long long epoch,
                                 unsigned long long limit_ns, cudaStream_t s) {
    k_wait_consumed<<<1, 64, 0, s>>>(mine, rank, p, epoch, limit_ns);
    return cudaGetLastError();
}

cudaError_t launch_pull_publish(P2PFlags *const *peer_flags, int rank, int p,
                                unsigned long long epoch, cudaStream_t s) {
    return launch_pdl(k_pull_publish, dim3(1), dim3(64), 0, s, peer_flags, rank, p, epoch);
}

cudaError_t launch_pull_wait(P2PFlags *mine, int rank, int p, unsigned long long epoch,
                             cudaStream_t s) {
    return launch_pdl(k_pull_wait, dim3(1), dim3(64), 0, s, mine, rank, p, epoch);
}

cudaError_t launch_p2p_push(const uint8_t *msg, uint8_t *const *stage, P2PFlags *const *peer_flags,
                            P2PFlags *mine, int rank, int p, unsigned long long epoch,
                            uint64_t msg_bytes, int L, uint32_t hdr_words, int nb, cudaStream_t s,
                            uint64_t tab_off, uint64_t tab_bytes) {
    return launch_pdl(k_p2p_push, dim3(nb, p), dim3(kThreads), 0, s, msg, stage, peer_flags, mine,
                      rank, p, epoch, msg_bytes, L, hdr_words, tab_off, tab_bytes);
}


}  // namespace rgc
