// pack.cu -- §8(a) step 2: validate each raw set and derive its analysis record (one warp per set).
//
// Reads the paper's system model from the flat CSR batch, checks the validation rules in
// the order documented in include/paam.h, and derives everything the fixed-point kernels
// need, so that they touch only integer arrays in shared memory:
//   * chain ranks (rank 0 = highest unique priority) and per-period mu constants (Eq.2);
//   * sub-chains = maximal runs of consecutive callbacks on one executor;
//   * E_i per callback, calligraphic E_c per sub-chain;
//   * A* = A + 2 kappa_eff with kappa_eff = 0 on a one-bucket accelerator (A6);
//   * the bucket of every (chain, accelerator): rank-based groups of ceil(m_a / n) (A5);
//   * LP blocking per segment: max A* of lower-priority segments in the same bucket and unit;
//   * W[u][k] = sum of A* of chain k on unit u (exact regrouping of the hps sums of Eq.3 / Eq.4);
//   * B_c as written, hp / hpp / lp sets as bit masks;
//   * the canonical analysis order: per core, process priority desc, then chain priority desc (A7).
// Lanes run over chains / callbacks / segments / sub-chains; all staging is in shared memory.
#include "common.cuh"

namespace paam {

namespace {

constexpr int WARPS = 4;
constexpr int MAXG = 192;  // segments per set

struct Scratch {
  uint32_t cT[MAXC], cD[MAXC], cPrio[MAXC], cCb0[MAXC];
  uint8_t cNcb[MAXC], cCls[MAXC], cRank[MAXC], cNsub[MAXC];
  uint32_t cUse[MAXC];  // bit a: chain uses accelerator a
  uint8_t cBucket[MAXC][4];
  uint32_t bSeg0[MAXCB], bE[MAXCB];
  uint8_t bNseg[MAXCB], bExec[MAXCB], bChain[MAXCB], bSub[MAXCB];
  uint32_t gW[MAXG];
  uint8_t gKind[MAXG], gAcc[MAXG], gUnit[MAXG], gCb[MAXG];
  uint32_t xPrio[MAXX];
  uint8_t xCore[MAXX], xWait[MAXX];
  uint32_t aN[4], aUnits[4], aUbase[4], aEps[4], aKeff[4], aServer[4];
  uint32_t qAstar[MAXA], qLPB[MAXA];
  uint8_t qChain[MAXA], qCb[MAXA], qSub[MAXA], qUnit[MAXA], qAcc[MAXA], qPos[MAXA];
  uint8_t uChain[MAXS], uExec[MAXS], uCb0[MAXS], uNcb[MAXS], uCanon[MAXS], uNa[MAXS], uA0[MAXS];
  unsigned long long W64[MAXU][MAXC];
};

__device__ __forceinline__ bool warp_any(bool p) { return __any_sync(0xffffffffu, p); }

__global__ void __launch_bounds__(WARPS * 32) pack_kernel(paam_batch b, Record* __restrict__ recs,
                                                          int32_t* __restrict__ status_out) {
  __shared__ Scratch smem[WARPS];
  const int lane = threadIdx.x & 31;
  Scratch& s = smem[threadIdx.x >> 5];
  const uint32_t nwarps = gridDim.x * WARPS;
  for (uint32_t set = blockIdx.x * WARPS + (threadIdx.x >> 5); set < b.n_sets; set += nwarps) {
    Record* r = recs + set;
    const uint32_t c0 = b.set_chain_off[set], c1 = b.set_chain_off[set + 1];
    const uint32_t x0 = b.set_exec_off[set], x1 = b.set_exec_off[set + 1];
    const uint32_t a0 = b.set_accel_off[set], a1 = b.set_accel_off[set + 1];
    const uint32_t nch = c1 - c0, nex = x1 - x0, nac = a1 - a0;
    const uint32_t cb0 = b.chain_cb_off[c0], cb1 = b.chain_cb_off[c1];
    const uint32_t ncb = cb1 - cb0;
    const uint32_t sg0 = b.cb_seg_off[cb0], sg1 = b.cb_seg_off[cb1];
    const uint32_t nseg = sg1 - sg0;
    int st = PAAM_SET_OK;
    uint32_t n_aseg = 0, n_sub = 0, n_unit = 0;

    // ---- 1. ERANGE: size caps, accelerator parameters, 31-bit times ------------------------------
    if (nch > MAXC || ncb > MAXCB || nseg > MAXG || nex > MAXX || nac > 4) st = PAAM_SET_ERANGE;
    if (st == PAAM_SET_OK) {
      bool bad = false;
      for (uint32_t base = 0; base < nseg; base += 32) {  // warp-uniform trip count (ballot)
        const uint32_t k = base + lane;
        uint8_t kind = 0;
        if (k < nseg) {
          kind = b.seg_kind[sg0 + k];
          const uint64_t w = b.seg_wcet[sg0 + k];
          s.gKind[k] = kind;
          s.gW[k] = (uint32_t)min(w, (uint64_t)SAT);
          s.gAcc[k] = b.seg_accel[sg0 + k];
          s.gUnit[k] = b.seg_unit[sg0 + k];
          bad |= (w >= LIM);
        }
        n_aseg += __popc(__ballot_sync(0xffffffffu, k < nseg && kind == 1));
      }
      for (uint32_t k = lane; k < nch; k += 32) {
        const uint64_t T = b.chain_T[c0 + k], D = b.chain_D[c0 + k];
        bad |= (T == 0 || T >= LIM || D >= LIM);
        s.cT[k] = (uint32_t)min(T, (uint64_t)SAT);
        s.cD[k] = (uint32_t)min(D, (uint64_t)SAT);
        s.cPrio[k] = b.chain_prio[c0 + k];
        s.cCls[k] = b.chain_class[c0 + k];
        s.cCb0[k] = b.chain_cb_off[c0 + k] - cb0;
        s.cNcb[k] = (uint8_t)min(b.chain_cb_off[c0 + k + 1] - b.chain_cb_off[c0 + k], 255u);
      }
      if (lane < nac) {
        const uint32_t n = b.accel_buckets[a0 + lane], u = b.accel_units[a0 + lane];
        const uint64_t e = b.accel_eps[a0 + lane], kp = b.accel_kappa[a0 + lane];
        bad |= (n < 1 || n > 32 || u < 1 || u > 8 || e >= LIM || kp >= LIM);
        s.aN[lane] = n;
        s.aUnits[lane] = u;
        s.aEps[lane] = (uint32_t)min(e, (uint64_t)SAT);
        s.aKeff[lane] = n > 1 ? (uint32_t)min(kp, (uint64_t)SAT) : 0u;  // A6
        s.aServer[lane] = b.accel_server_core[a0 + lane];
      }
      __syncwarp();
      if (lane == 0) {
        uint32_t ub = 0;
        for (uint32_t a = 0; a < nac; a++) { s.aUbase[a] = ub; ub += s.aUnits[a]; }
        n_unit = ub;
      }
      n_unit = __shfl_sync(0xffffffffu, n_unit, 0);
      if (warp_any(bad) || n_aseg > MAXA || n_unit > MAXU) st = PAAM_SET_ERANGE;
    }
    if (st == PAAM_SET_OK) {
      for (uint32_t k = lane; k < ncb; k += 32) {
        const uint32_t so = b.cb_seg_off[cb0 + k];
        s.bSeg0[k] = so - sg0;
        s.bNseg[k] = (uint8_t)min(b.cb_seg_off[cb0 + k + 1] - so, 255u);
        s.bExec[k] = (uint8_t)min((uint32_t)b.cb_exec[cb0 + k], 255u);
      }
      for (uint32_t k = lane; k < nex; k += 32) {
        s.xCore[k] = b.exec_core[x0 + k];
        s.xPrio[k] = b.exec_prio[x0 + k];
        s.xWait[k] = b.exec_wait[x0 + k];
      }
      __syncwarp();
      // callback -> chain, segment -> callback
      for (uint32_t c = lane; c < nch; c += 32)
        for (uint32_t j = 0; j < s.cNcb[c]; j++) s.bChain[s.cCb0[c] + j] = (uint8_t)c;
      for (uint32_t j = lane; j < ncb; j += 32)
        for (uint32_t k = 0; k < s.bNseg[j]; k++) s.gCb[s.bSeg0[j] + k] = (uint8_t)j;
      __syncwarp();
      // ---- 2. EDANGLING ---------------------------------------------------------------------------
      bool bad = false;
      for (uint32_t c = lane; c < nch; c += 32) bad |= (s.cNcb[c] == 0);
      for (uint32_t j = lane; j < ncb; j += 32) bad |= (s.bNseg[j] == 0 || s.bExec[j] >= nex);
      for (uint32_t k = lane; k < nseg; k += 32)
        bad |= (s.gKind[k] == 1 && s.gAcc[k] < nac && s.gUnit[k] >= s.aUnits[s.gAcc[k]]);
      if (warp_any(bad)) st = PAAM_SET_EDANGLING;
    }
    if (st == PAAM_SET_OK) {  // ---- 3. EACCEL ---------------------------------------------------
      bool bad = false;
      for (uint32_t k = lane; k < nseg; k += 32) bad |= (s.gKind[k] == 1 && s.gAcc[k] >= nac);
      if (warp_any(bad)) st = PAAM_SET_EACCEL;
    }
    if (st == PAAM_SET_OK) {  // ---- 4. ESHAPE ---------------------------------------------------
      bool bad = false;
      for (uint32_t x = lane; x < nex; x += 32) bad |= (s.xWait[x] > 1);
      for (uint32_t c = lane; c < nch; c += 32) bad |= (s.cCls[c] > 1);
      for (uint32_t k = lane; k < nseg; k += 32) {
        bad |= (s.gKind[k] > 1 || s.gW[k] == 0);
        if (k > 0 && s.gCb[k - 1] == s.gCb[k]) bad |= (s.gKind[k] == s.gKind[k - 1]);
      }
      for (uint32_t j = lane; j < ncb; j += 32) {  // a chain never re-enters an executor (A13)
        const uint32_t c = s.bChain[j], f = s.cCb0[c];
        if (j > f && s.bExec[j] != s.bExec[j - 1])
          for (uint32_t i = f; i + 1 < j; i++) bad |= (s.bExec[i] == s.bExec[j]);
      }
      if (warp_any(bad)) st = PAAM_SET_ESHAPE;
    }
    if (st == PAAM_SET_OK) {  // ---- 4b. sub-chains and their count ---------------------------------
      for (uint32_t base = 0; base < ncb; base += 32) {
        const uint32_t j = base + lane;
        bool start = false;
        if (j < ncb) start = (j == s.cCb0[s.bChain[j]]) || (s.bExec[j] != s.bExec[j - 1]);
        n_sub += __popc(__ballot_sync(0xffffffffu, start));
      }
      // sub-chain id of a callback = (number of run starts up to and including it) - 1
      for (uint32_t j = lane; j < ncb; j += 32) {
        uint32_t cnt = 0;
        for (uint32_t i = 0; i <= j; i++)
          cnt += (i == s.cCb0[s.bChain[i]]) || (s.bExec[i] != s.bExec[i - 1]);
        s.bSub[j] = (uint8_t)min(cnt - 1, 255u);
      }
      if (n_sub > MAXS) st = PAAM_SET_ERANGE;
    }
    if (st == PAAM_SET_OK) {  // ---- 5. EDUPPRIO --------------------------------------------------
      bool bad = false;
      for (uint32_t c = lane; c < nch; c += 32)
        for (uint32_t d = 0; d < nch; d++) bad |= (d != c && s.cPrio[d] == s.cPrio[c]);
      for (uint32_t x = lane; x < nex; x += 32)
        for (uint32_t y = 0; y < nex; y++) bad |= (y != x && s.xCore[y] == s.xCore[x] && s.xPrio[y] == s.xPrio[x]);
      if (warp_any(bad)) st = PAAM_SET_EDUPPRIO;
    }
    if (st == PAAM_SET_OK) {  // ---- 6. EDEADLINE -------------------------------------------------
      bool bad = false;
      for (uint32_t c = lane; c < nch; c += 32) bad |= (s.cD[c] == 0 || (s.cCls[c] == 0 && s.cD[c] > s.cT[c]));
      if (warp_any(bad)) st = PAAM_SET_EDEADLINE;
    }
    if (st == PAAM_SET_OK) {  // ---- 7. ECORE (R1) ------------------------------------------------
      bool bad = false;
      for (uint32_t x = lane; x < nex; x += 32)
        for (uint32_t a = 0; a < nac; a++) bad |= (s.xCore[x] == s.aServer[a]);
      if (warp_any(bad)) st = PAAM_SET_ECORE;
    }

    if (lane == 0) {
      r->status = st;
      r->chain_base = c0;
      r->bin = b.set_bin ? b.set_bin[set] : 0u;
      r->n_out = nch;
    }
    if (status_out && lane == 0) status_out[set] = st;
    if (st != PAAM_SET_OK) {
      if (lane == 0) { r->n_chain = 0; r->n_sub = 0; r->n_aseg = 0; r->n_unit = 0; }
      __syncwarp();
      continue;
    }

    // ======================== derivation (valid set) ==================================================
    // chain ranks: number of chains with a higher priority (priorities are unique)
    for (uint32_t c = lane; c < nch; c += 32) {
      uint32_t rk = 0;
      for (uint32_t d = 0; d < nch; d++) rk += (s.cPrio[d] > s.cPrio[c]);
      s.cRank[c] = (uint8_t)rk;
      s.cUse[c] = 0;
      s.cNsub[c] = 0;
    }
    // E_i of each callback: its CPU segments, saturating
    for (uint32_t j = lane; j < ncb; j += 32) {
      uint32_t e = 0;
      for (uint32_t k = 0; k < s.bNseg[j]; k++)
        if (s.gKind[s.bSeg0[j] + k] == 0) e = sadd(e, s.gW[s.bSeg0[j] + k]);
      s.bE[j] = e;
    }
    for (uint32_t i = lane; i < MAXU * MAXC; i += 32) (&s.W64[0][0])[i] = 0ull;
    __syncwarp();
    // accelerator segments in original order: compaction by ballot
    {
      uint32_t q0 = 0;
      for (uint32_t base = 0; base < nseg; base += 32) {
        const uint32_t k = base + lane;
        const bool isA = (k < nseg) && s.gKind[k] == 1;
        const uint32_t bal = __ballot_sync(0xffffffffu, isA);
        if (isA) {
          const uint32_t q = q0 + __popc(bal & ((1u << lane) - 1u));
          const uint32_t j = s.gCb[k], c = s.bChain[j], a = s.gAcc[k];
          s.qChain[q] = (uint8_t)c;
          s.qCb[q] = (uint8_t)j;
          s.qSub[q] = s.bSub[j];
          s.qAcc[q] = (uint8_t)a;
          s.qUnit[q] = (uint8_t)(s.aUbase[a] + s.gUnit[k]);
          s.qAstar[q] = sadd(s.gW[k], sadd(s.aKeff[a], s.aKeff[a]));  // A* = A + 2 kappa_eff
          atomicOr(&s.cUse[c], 1u << a);
        }
        q0 += __popc(bal);
      }
    }
    __syncwarp();
    // buckets (A5): per accelerator, users ranked by priority, groups of ceil(m_a / n)
    for (uint32_t a = 0; a < nac; a++) {
      const bool use = (lane < nch) && ((s.cUse[lane] >> a) & 1u);
      const uint32_t ma = __popc(__ballot_sync(0xffffffffu, use));
      if (lane < nch) {
        uint32_t ra = 0;
        for (uint32_t d = 0; d < nch; d++) ra += ((s.cUse[d] >> a) & 1u) && s.cRank[d] < s.cRank[lane];
        const uint32_t n = s.aN[a], g = (ma + n - 1) / n;
        s.cBucket[lane][a] = use ? (uint8_t)(n - 1 - ra / g) : 0xFF;
      }
    }
    __syncwarp();
    // LP blocking and regrouped weights W
    for (uint32_t q = lane; q < n_aseg; q += 32) {
      const uint32_t c = s.qChain[q], u = s.qUnit[q], a = s.qAcc[q];
      const uint32_t bk = s.cBucket[c][a];
      uint32_t lpb = 0;
      for (uint32_t p = 0; p < n_aseg; p++) {
        const uint32_t d = s.qChain[p];
        if (s.qUnit[p] == u && s.cRank[d] > s.cRank[c] && s.cBucket[d][a] == bk) lpb = max(lpb, s.qAstar[p]);
      }
      s.qLPB[q] = lpb;
      atomicAdd(&s.W64[u][s.cRank[c]], (unsigned long long)s.qAstar[q]);
    }
    // sub-chain table in original order
    for (uint32_t j = lane; j < ncb; j += 32) {
      const bool start = (j == s.cCb0[s.bChain[j]]) || (s.bExec[j] != s.bExec[j - 1]);
      if (start) {
        const uint32_t u = s.bSub[j];
        uint32_t n = 1;
        while (j + n < ncb && s.bSub[j + n] == u) n++;
        s.uChain[u] = s.bChain[j];
        s.uExec[u] = s.bExec[j];
        s.uCb0[u] = (uint8_t)j;
        s.uNcb[u] = (uint8_t)n;
      }
    }
    __syncwarp();
    // canonical order (A7): per core, process priority desc, chain rank asc
    for (uint32_t u = lane; u < n_sub; u += 32) {
      const uint32_t xu = s.uExec[u], ru = s.cRank[s.uChain[u]];
      const uint32_t cu = s.xCore[xu], pu = s.xPrio[xu];
      uint32_t pos = 0;
      for (uint32_t v = 0; v < n_sub; v++) {
        const uint32_t xv = s.uExec[v], rv = s.cRank[s.uChain[v]];
        const uint32_t cv = s.xCore[xv], pv = s.xPrio[xv];
        pos += (cv < cu) || (cv == cu && (pv > pu || (pv == pu && rv < ru)));
      }
      s.uCanon[u] = (uint8_t)pos;
      uint32_t na = 0;
      for (uint32_t q = 0; q < n_aseg; q++) na += (s.qSub[q] == u);
      s.uNa[u] = (uint8_t)na;
    }
    __syncwarp();
    // first accelerator segment of each sub-chain in canonical grouping
    for (uint32_t u = lane; u < n_sub; u += 32) {
      uint32_t f = 0;
      for (uint32_t v = 0; v < n_sub; v++) f += (s.uCanon[v] < s.uCanon[u]) ? s.uNa[v] : 0u;
      s.uA0[u] = (uint8_t)f;
    }
    __syncwarp();
    for (uint32_t q = lane; q < n_aseg; q += 32) {
      const uint32_t u = s.qSub[q];
      uint32_t k = 0;
      for (uint32_t p = 0; p < q; p++) k += (s.qSub[p] == u);
      s.qPos[q] = (uint8_t)(s.uA0[u] + k);
    }
    __syncwarp();

    // ---- write the record ---------------------------------------------------------------------------
    if (lane == 0) { r->n_chain = (uint8_t)nch; r->n_sub = (uint8_t)n_sub; r->n_aseg = (uint8_t)n_aseg; r->n_unit = (uint8_t)n_unit; }
    // chains by rank
    for (uint32_t c = lane; c < nch; c += 32) {
      const uint32_t k = s.cRank[c];
      uint32_t M, L;
      make_magic(s.cT[c], &M, &L);
      uint32_t nsub = 0;
      for (uint32_t u = 0; u < n_sub; u++) nsub += (s.uChain[u] == c);
      r->cT[k] = s.cT[c];
      r->cCut[k] = min(s.cD[c], s.cT[c]);
      r->cD[k] = s.cD[c];
      r->cM[k] = M;
      r->cMisc[k] = L | ((uint32_t)s.cCls[c] << 8) | (c << 16) | (nsub << 24);
    }
    for (uint32_t i = lane; i < n_unit * MAXC; i += 32) {
      const uint32_t u = i / MAXC, k = i % MAXC;
      const unsigned long long w = s.W64[u][k];
      r->W[u][k] = w > SAT ? SAT : (uint32_t)w;
    }
    // sub-chains in canonical order
    for (uint32_t u = lane; u < n_sub; u += 32) {
      const uint32_t c = s.uChain[u], x = s.uExec[u], rk = s.cRank[c];
      uint32_t E = 0;
      for (uint32_t j = s.uCb0[u]; j < s.uCb0[u] + s.uNcb[u]; j++) E = sadd(E, s.bE[j]);
      uint32_t eps = 0, base3 = 0, umask = 0;
      for (uint32_t q = 0; q < n_aseg; q++)
        if (s.qSub[q] == u) {
          eps = sadd(eps, s.aEps[s.qAcc[q]]);
          base3 = sadd(base3, sadd(s.qAstar[q], s.qLPB[q]));
          umask |= 1u << s.qUnit[q];
        }
      uint32_t B = 0;  // B_c = max E_j over callbacks of lower-priority chains on the executor
      for (uint32_t j = 0; j < ncb; j++)
        if (s.bExec[j] == x && s.cRank[s.bChain[j]] > rk) B = max(B, s.bE[j]);
      uint32_t hp = 0, hpp = 0, lp = 0;
      for (uint32_t v = 0; v < n_sub; v++) {
        const uint32_t xv = s.uExec[v], rv = s.cRank[s.uChain[v]];
        const uint32_t bit = 1u << s.uCanon[v];
        if (v == u) continue;
        if (xv == x) {
          if (rv < rk) hp |= bit;
          else lp |= bit;
        } else if (s.xCore[xv] == s.xCore[x] && s.xPrio[xv] > s.xPrio[x]) {
          hpp |= bit;
        }
      }
      uint32_t pos = 0;  // position of the sub-chain inside its chain
      for (uint32_t v = 0; v < u; v++) pos += (s.uChain[v] == c);
      const uint32_t k = s.uCanon[u];
      r->sE[k] = E;
      r->sB[k] = B;
      r->sEps[k] = eps;
      r->sBase3[k] = base3;
      r->sHp[k] = hp;
      r->sHpp[k] = hpp;
      r->sLp[k] = lp;
      r->sMisc[k] = rk | (umask << 8) | ((uint32_t)(s.xWait[x] == 1) << 16) | (pos << 24);
      r->sSeg[k] = (uint32_t)s.uA0[u] | ((uint32_t)s.uNa[u] << 8) | (x << 16) | ((uint32_t)s.xCore[x] << 24);
    }
    // accelerator segments grouped by canonical sub-chain
    for (uint32_t q = lane; q < n_aseg; q += 32) {
      const uint32_t p = s.qPos[q];
      const uint32_t c = s.qChain[q];
      r->aBase2[p] = sadd(s.qAstar[q], s.qLPB[q]);
      r->aEps[p] = s.aEps[s.qAcc[q]];
      r->aCbE[p] = s.bE[s.qCb[q]];
      r->aMisc[p] = (uint32_t)s.cRank[c] | ((uint32_t)s.qUnit[q] << 8) | ((uint32_t)s.uCanon[s.qSub[q]] << 16) |
                    ((uint32_t)s.qCb[q] << 24);
    }
    __syncwarp();
  }
}

}  // namespace

int launch_pack(const paam_batch* b, Record* rec, int32_t* status, cudaStream_t st) {
  if (b->n_sets == 0) return PAAM_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t need = (b->n_sets + WARPS - 1) / WARPS;
  const uint32_t grid = need < (uint32_t)sms * 16 ? need : (uint32_t)sms * 16;
  pack_kernel<<<grid, WARPS * 32, 0, st>>>(*b, rec, status);
  count_launch();
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? PAAM_OK : fail_cuda(e, "pack_kernel launch");
}

}  // namespace paam
