/*
 * Schedule-sensitivity experiments (TEST INFRASTRUCTURE, not the product and not a pin):
 * replays of other schedules of the same coordinate steps, built on the oracle's own step
 * functions (it includes oracle/thetis_ref.c), to measure how far each schedule moves the
 * 20-epoch point from Alg. 1's permuted sweep (oracle MODE_ASYNC).  Used by
 * tests/experiments/schedule_sensitivity.py; results in profiles/r02_schedule_sensitivity.txt.
 */
#include "../../oracle/thetis_ref.c"

/* the permuted sweep over all tiles in windows of W consecutive positions: every unit of a
 * window steps from the window's start state (a pessimistic model of W tiles in flight);
 * slack_first: all slacks step first in each epoch (sequentially), then the window sweep
 * skips them.  W = 1 with slack_first = 0 is mode 4 without the block / scalar / slack groups. */
int exp_window(ref_lp* lp, float beta, int epochs, uint64_t seed, int rule, int64_t W, int slack_first) {
    step_ctx s = make_ctx(lp, beta, rule);
    int64_t n_tiles = (lp->U + 31) / 32, nsu = lp->n_blocks + lp->n_scalar;
    int64_t kk = lp->block_k > 0 ? lp->block_k : 1;
    int64_t* perm = (int64_t*)xcalloc(n_tiles, sizeof(int64_t));
    REAL* nv = (REAL*)xcalloc(W * 32 * kk, sizeof(REAL));
    int64_t* us = (int64_t*)xcalloc(W * 32, sizeof(int64_t));
    for (int e = 0; e < epochs; e++) {
        thetis_ref_tile_perm(n_tiles, seed, e, perm);
        if (slack_first)
            for (int64_t u = nsu; u < lp->U; u++) step_unit(lp, &s, u);
        for (int64_t t0 = 0; t0 < n_tiles; t0 += W) {
            int64_t cnt = 0;
            for (int64_t t = t0; t < t0 + W && t < n_tiles; t++)
                for (int64_t u = perm[t] * 32; u < perm[t] * 32 + 32 && u < lp->U; u++) {
                    if (unit_fixed(lp, u) || (slack_first && u >= nsu)) continue;
                    unit_new_values(lp, &s, u, nv + cnt * kk);
                    us[cnt++] = u;
                }
            for (int64_t q = 0; q < cnt; q++) apply_unit(lp, us[q], nv + q * kk);
        }
    }
    free(perm); free(nv); free(us);
    return 0;
}

/* hub schedules after a slack-first sweep (hub tile = scalar tile with > hub_nnz nonzeros):
 *   0: hubs one at a time (fresh r) in permuted order before the light tiles
 *   1: hubs one synchronous step from the post-slack state, applied at once
 *   2: hubs one synchronous step, applied after the light tiles (the hub-lag idea)
 *   3: hubs in their permuted position with the light tiles (only the slacks moved) */
int exp_hubs(ref_lp* lp, float beta, int epochs, uint64_t seed, int rule, int sched, int64_t hub_nnz) {
    step_ctx s = make_ctx(lp, beta, rule);
    int64_t nsu = lp->n_blocks + lp->n_scalar, nst = (nsu + 31) / 32;
    int64_t* perm = (int64_t*)xcalloc(nst, sizeof(int64_t));
    uint8_t* hub = (uint8_t*)xcalloc(nst, 1);
    for (int64_t t = 0; t < nst; t++) {
        int64_t nz = 0;
        for (int64_t u = t * 32; u < t * 32 + 32 && u < nsu; u++) nz += col_nnz(lp, u);
        hub[t] = nz > hub_nnz;
    }
    REAL* nv = (REAL*)xcalloc(nsu + 1, sizeof(REAL));
    for (int e = 0; e < epochs; e++) {
        for (int64_t u = nsu; u < lp->U; u++) step_unit(lp, &s, u);
        thetis_ref_tile_perm(nst, seed, e, perm);
        if (sched == 0) {
            for (int64_t t = 0; t < nst; t++)
                if (hub[perm[t]])
                    for (int64_t u = perm[t] * 32; u < perm[t] * 32 + 32 && u < nsu; u++) step_unit(lp, &s, u);
        } else if (sched == 1 || sched == 2) {
            for (int64_t t = 0; t < nst; t++)
                if (hub[t])
                    for (int64_t u = t * 32; u < t * 32 + 32 && u < nsu; u++) unit_new_values(lp, &s, u, nv + u);
            if (sched == 1)
                for (int64_t t = 0; t < nst; t++)
                    if (hub[t])
                        for (int64_t u = t * 32; u < t * 32 + 32 && u < nsu; u++) apply_unit(lp, u, nv + u);
        }
        for (int64_t t = 0; t < nst; t++) {
            if (sched != 3 && hub[perm[t]]) continue;
            for (int64_t u = perm[t] * 32; u < perm[t] * 32 + 32 && u < nsu; u++) step_unit(lp, &s, u);
        }
        if (sched == 2)
            for (int64_t t = 0; t < nst; t++)
                if (hub[t])
                    for (int64_t u = t * 32; u < t * 32 + 32 && u < nsu; u++) apply_unit(lp, u, nv + u);
    }
    free(perm); free(hub); free(nv);
    return 0;
}

/* grouped hub schedule (after a slack-first sweep): structural unit u belongs to group grp[u]
 * in [0, G) or is light (grp[u] < 0).  Per epoch the groups come in the order of a Fisher-Yates
 * shuffle from SplitMix64(seed, e) when permute != 0 (else 0..G-1); the units of a group take one
 * synchronous step from the state left by the earlier groups (Jacobi inside a group, Gauss-Seidel
 * across groups); then the light tiles in the permuted order, one unit at a time.
 * jacobi_in_group = 0 makes the units of a group step one at a time too (the sequential order
 * the grouped schedule approximates). */
static uint64_t sv_mix(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
int exp_groups(ref_lp* lp, float beta, int epochs, uint64_t seed, int rule, const int32_t* grp, int G, int permute,
               int jacobi_in_group) {
    step_ctx s = make_ctx(lp, beta, rule);
    int64_t nsu = lp->n_blocks + lp->n_scalar, nst = (nsu + 31) / 32;
    int64_t* perm = (int64_t*)xcalloc(nst, sizeof(int64_t));
    REAL* nv = (REAL*)xcalloc(nsu + 1, sizeof(REAL));
    /* members of each group, ascending */
    int64_t* cnt = (int64_t*)xcalloc(G + 1, sizeof(int64_t));
    for (int64_t u = 0; u < nsu; u++) if (grp[u] >= 0) cnt[grp[u] + 1]++;
    for (int g = 0; g < G; g++) cnt[g + 1] += cnt[g];
    int64_t* mem = (int64_t*)xcalloc(cnt[G] + 1, sizeof(int64_t));
    int64_t* fill = (int64_t*)xcalloc(G + 1, sizeof(int64_t));
    for (int64_t u = 0; u < nsu; u++) if (grp[u] >= 0) mem[cnt[grp[u]] + fill[grp[u]]++] = u;
    int* order = (int*)xcalloc(G + 1, sizeof(int));
    for (int e = 0; e < epochs; e++) {
        for (int64_t u = nsu; u < lp->U; u++) step_unit(lp, &s, u);
        for (int g = 0; g < G; g++) order[g] = g;
        if (permute) {
            uint64_t st = sv_mix(seed ^ (0xA0761D6478BD642Full * (uint64_t)(e + 1)));
            for (int g = G - 1; g > 0; g--) {
                st = sv_mix(st);
                int j = (int)(st % (uint64_t)(g + 1));
                int t = order[g]; order[g] = order[j]; order[j] = t;
            }
        }
        for (int q = 0; q < G; q++) {
            int g = order[q];
            if (jacobi_in_group) {
                for (int64_t i = cnt[g]; i < cnt[g + 1]; i++) unit_new_values(lp, &s, mem[i], nv + mem[i]);
                for (int64_t i = cnt[g]; i < cnt[g + 1]; i++) apply_unit(lp, mem[i], nv + mem[i]);
            } else {
                for (int64_t i = cnt[g]; i < cnt[g + 1]; i++) step_unit(lp, &s, mem[i]);
            }
        }
        thetis_ref_tile_perm(nst, seed, e, perm);
        for (int64_t t = 0; t < nst; t++)
            for (int64_t u = perm[t] * 32; u < perm[t] * 32 + 32 && u < nsu; u++)
                if (grp[u] < 0) step_unit(lp, &s, u);
    }
    free(perm); free(nv); free(cnt); free(mem); free(fill); free(order);
    return 0;
}
