// chain.cu — K_chain: stage 2 (merge of a survivor's per-tile partials in tile
// order, backward.hpp:141-145) and stage 3 (camera / world chain,
// backward.hpp:148-185, grad_chain.hpp:48-77) in the inverse-free fp32 closed
// form, one thread per survivor, CTA per K_decide group. Built with FMA
// contraction; the fp64-decided survivors take K_chain_exact (prep.cu).
#include "chain.cuh"
#include "common.cuh"
#include "focus.cuh"

namespace gpk {

namespace {

// K_chain: one thread per survivor (backward.hpp:148-185). Survivors that
// fast_prepare resolves (the same decision K_exact made: identical code and
// inputs) take the inverse-free fp32 chain; the rest are deferred to
// K_chain_exact so this kernel stays small in registers.
__global__ void __launch_bounds__(256) k_chain(const ChainLaunch a) {
    pdl_entry();  // see common.cuh: successor may launch; predecessor complete
    // CTA per K_decide group: its survivors sit at slots [g*4096, g*4096 + S_g)
    const unsigned g = blockIdx.x;
    const unsigned S = a.grp_surv[g];
    const bool dense = a.slot_grads == nullptr;  // dense planes: keep the sparse-clear list
    if (dense && g == 0 && threadIdx.x == 0) *a.grads_dirty = a.ctrl->survivors;
    for (unsigned j = threadIdx.x; j < S; j += blockDim.x) {
        const uint32_t cid = g * kDecideGroupSize + j;
        // the record and the parameters requested together (the branch on the
        // record would otherwise hold the parameters' load for a round trip)
        const SurvivorRecord rec = a.records[cid];
        float pf[11];
        uint32_t i;
        load_cand(a.sparams + cid, pf, i);
        if (dense) a.dirty_idx[atomicAdd(a.dirty_ctr, 1u)] = rec.gidx & ~kExactFlag;
        if (rec.gidx & kExactFlag) continue;  // K_chain_exact (listed by K_decide)
        PartialsBatch pb;  // the partials' loads overlap the forward state's arithmetic
        merge_partials_issue(a, rec, pb);
        FastFocus ff;
        fast_state(pf, a.slice, ff);
        double acc[6];
        merge_partials_finish(pb, acc);
        float g11[11], dmu[3];
        fast_backward(pf, ff, acc, a.slice, g11, dmu);
        store_chain(a, i, cid, g11, dmu, acc);
    }
}

}  // namespace

void launch_chain(const ChainLaunch& a, int grid, int num_sms, cudaStream_t st) {
    // CTA per group; more groups than one wave of 256-thread CTAs (3 per SM):
    // 128 threads (a group holds ~100-200 survivors: more CTAs in flight)
    const int threads = grid > 3 * num_sms ? 128 : 256;
    launch_pdl(k_chain, dim3(grid), dim3(threads), 0, st, a);
}

}  // namespace gpk
