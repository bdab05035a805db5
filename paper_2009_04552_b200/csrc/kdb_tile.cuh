// kdb_tile.cuh -- round 1 of the light rows-Boruvka as tile-local Boruvka in shared memory
// Part of kdb.cu's single translation unit: included inside its anonymous
// namespace, after kdb_rows.cuh; not a standalone header.
#pragma once

// ============================================================================
// Tile round (DESIGN.md §6 "Tile round").  The paper builds a LOCAL MST per
// process before any exchange (Alg. 2) on points partitioned
// so that a process's points are spatially compact; here the
// same idea runs one level down: a CTA takes a tile of kTileRows consecutive
// rows (a compact piece of the data set when the ids follow the partition),
// stages the tile's light ELL rows in shared memory and runs Boruvka rounds on
// the tile's components there, until no component of the tile can hook inside
// it.  Exactness is the rows-Boruvka's own argument (reading #20): a
// component's offer is the minimum over its rows' live entries -- entries
// leaving the TILE included -- and it hooks only along a certified minimum
// whose other end lies in the tile; a component whose minimum leaves the tile
// (or cannot be decided from the ELL) waits, and may still absorb components
// that hook into it (its minimum is then re-taken next round).  So every hook
// is along an edge of the exact MSF (the cut property under the strict order
// O1), mutual pairs resolve as in k_hook, and the global rounds continue from
// the contracted components with the rows still live and their heads.
//
// Outputs, as round 1 of rows_phase: parent[c] for every dense core id (the
// dense id of its in-tile root; depth <= 1), the MSF edges of the tile's hooks
// (e_key/e_w layout of k_hook), the live rows with their heads, and the
// counters (hooks, offered).  contract() then renumbers as after any round.
// rows per tile = threads per CTA (one row per thread): 1,024 (one CTA per SM)
// or 512 (two CTAs per SM: one stages its tile while the other runs rounds)
constexpr int kTileMaxRounds = 48;          // safety bound; tiles converge in ~log2(tile) rounds
constexpr int32_t kTgtOut = -2;             // the minimum leaves the tile or is undecidable in it
constexpr int kDead = -1, kOut = -2, kEnd = -3;  // entry codes (else: the target's row in the tile)

template <int kTileRows>
struct TileSmem {
  int2 E[kW * kTileRows];     // the tile's ELL, column-major: E[c * T + row] = (J, w bits)
  uint64_t K[kTileRows];      // per local root: minimum offered key
  uint64_t ekey[kTileRows];   // staged MSF edges: (b << 32) | w bits
  uint32_t ea[kTileRows];     //                    a
  int32_t cvd[kTileRows];     // dense core id of the row (-1: non-core)
  int32_t lc[kTileRows];      // local root (row index in the tile) of the row's component
  int32_t par[kTileRows];     // per local root: hook target this round
  int32_t tg[kTileRows];      // per local root: target of the minimum (kTgtOut: outside); then new root
  uint64_t BT[kTileRows];     // per local root: (b << 32 | target + 2), minimum among offers of key K
  uint32_t km[kTileRows];     // per local root: certificate bound (kmin, mono bits)
  int16_t code[kW * kTileRows];  // per ELL entry (column-major): target row in the tile, or kOut / kDead / kEnd
  uint32_t wcnt[kTileRows / 32];
  uint32_t tile, n_edges, edge_base, live_base;
};

template <int kTileRows>
__global__ void __launch_bounds__(kTileRows) k_tile_round(
    const int4* __restrict__ LE, int64_t n_rows, int32_t k, float eps, int64_t N,
    const int32_t* __restrict__ comp, const uint32_t* __restrict__ core_bits, const uint32_t* __restrict__ kmin,
    int32_t* __restrict__ parent,
    uint64_t* __restrict__ e_key, float* __restrict__ e_w, int64_t e_cap, Rec* __restrict__ act_out,
    uint32_t* __restrict__ n_out, uint32_t* __restrict__ grab, RoundCounters* __restrict__ ctr,
    unsigned long long* __restrict__ n_entries, int max_rounds) {
  extern __shared__ __align__(16) unsigned char tile_smem_raw[];
  TileSmem<kTileRows>& S = *reinterpret_cast<TileSmem<kTileRows>*>(tile_smem_raw);
  const int i = threadIdx.x;
  const int lane = i & 31, wid = i >> 5;
  uint32_t hooks = 0, offered = 0;
  unsigned long long reads = 0;
  for (;;) {
    if (i == 0) { S.tile = atomicAdd(grab, 1u); S.n_edges = 0; }
    __syncthreads();
    const int64_t r0 = (int64_t)S.tile * kTileRows;
    if (r0 >= n_rows) break;
    const int nr = (int)min((int64_t)kTileRows, n_rows - r0);
    {  // the tile's ELL rows (coalesced) into COLUMN-major
       // shared memory: E[c * T + row], so a warp's 32 rows read one column
       // without bank conflicts (row-major 128-B rows put them all in one bank)
      // plane p holds the rows' 32-B chunks p: the tile's part of a plane is
      // nr * 32 contiguous bytes
      for (int q = i; q < nr * (kW / 2); q += kTileRows) {
        const int p = q / (2 * nr), j = q - p * 2 * nr;
        const int4 x = __ldcs(LE + (int64_t)p * ell_ps(n_rows) + ell_row(r0 + (j >> 1)) + (j & 1));
        const int r = j >> 1, c = 4 * p + 2 * (j & 1);
        S.E[c * kTileRows + r] = make_int2(x.x, x.y);
        S.E[(c + 1) * kTileRows + r] = make_int2(x.z, x.w);
      }
    }
    const int64_t v = r0 + i;
    const int32_t cv = i < nr ? __ldg(comp + v) : -1;
    S.cvd[i] = cv;
    __syncthreads();  // the tile's ELL and core flags are staged
    if (cv >= 0) {
      // one code per entry, so the rounds below read shared memory only:
      // kEnd (w > eps: the sorted row ends), kDead (padding, self, non-core
      // target -- the core test of targets outside the tile once, from the
      // L2-resident core bits), kOut (a core vertex outside the tile: always
      // another component), else the target's row in the tile
      const int2* er = S.E + i;       // column c of row i at [c * T]
      int16_t* cr = S.code + i;
#pragma unroll
      for (int c = 0; c < kW; ++c) {
        const int2 e = er[c * kTileRows];
        const int32_t J = e.x;
        int cd;
        if (!(__int_as_float(e.y) <= eps)) cd = kEnd;
        else if (J < 0 || J >= N || J == v) cd = kDead;
        else if (J >= r0 && J < r0 + nr) cd = S.cvd[J - r0] >= 0 ? (int)(J - r0) : kDead;
        else cd = is_core(core_bits, J) ? kOut : kDead;
        cr[c * kTileRows] = (int16_t)cd;
      }
    }
    S.lc[i] = cv >= 0 ? i : -1;
    S.K[i] = kSent;
    S.BT[i] = ~0ull;
    S.tg[i] = -1;
    S.km[i] = cv >= 0 ? __ldg(kmin + cv) : kInfBits;
    bool live = cv >= 0;  // the row still has (or may have) a leaving light entry
    int head = 0;
    __syncthreads();
    for (int rr = 0; rr < max_rounds; ++rr) {
      // ---- offers: the row's first leaving entry group (ties on w), from its head
      uint64_t best = kSent;
      uint32_t bestb = kSentB;
      int32_t btg = -1;
      const int32_t myc = live ? S.lc[i] : -1;
      if (live) {
        const int16_t* cr = S.code + i;
        const int head0 = head;
        int c = head, fc = -1;
        int32_t t = -1;
        for (; c < kW; ++c) {  // dead entries before the first leaving one stay dead
          const int cd = cr[c * kTileRows];
          if (cd == kEnd) break;
          if (cd == kDead) { head = c + 1; continue; }
          t = cd == kOut ? kTgtOut : S.lc[cd];
          if (t == myc) { head = c + 1; continue; }  // intra: dead for good (components only grow)
          fc = c;
          break;
        }
        reads += (unsigned long long)(min(c + 1, kW) - head0);
        bool open_end = false;  // the decision may depend on entries past the ELL
        if (fc >= 0) {
          const int2 e = S.E[fc * kTileRows + i];
          const uint32_t wstar = mono_bits(__int_as_float(e.y));
          const uint32_t vu = (uint32_t)v;
          best = pack_key(wstar, min(vu, (uint32_t)e.x));
          bestb = max(vu, (uint32_t)e.x);
          btg = t;
          int c2 = fc + 1;
          for (; c2 < kW; ++c2) {  // the tie group of the minimum's weight
            const int2 e2 = S.E[c2 * kTileRows + i];
            if (mono_bits(__int_as_float(e2.y)) != wstar) break;
            const int cd = cr[c2 * kTileRows];
            if (cd < 0 && cd != kOut) continue;
            const int32_t t2 = cd == kOut ? kTgtOut : S.lc[cd];
            if (t2 == myc) continue;
            const uint64_t kk = pack_key(wstar, min(vu, (uint32_t)e2.x));
            const uint32_t bb = max(vu, (uint32_t)e2.x);
            if (kk < best || (kk == best && bb < bestb)) { best = kk; bestb = bb; btg = t2; }
          }
          open_end = c2 == kW;
        } else {
          open_end = c == kW;  // every ELL entry is within eps and dead
        }
        if (open_end && k > kW) {
          // the candidate prefix (or the minimum's tie group) runs past the ELL:
          // the row's next entries are unknown here -- a lower bound (w of the
          // last ELL entry, a = b = 0, below every real key of that weight)
          // keeps the component from hooking on anything heavier
          best = pack_key(mono_bits(__int_as_float(S.E[(kW - 1) * kTileRows + i].y)), 0u);
          bestb = 0u;
          btg = kTgtOut;
        } else if (fc < 0) {
          live = false;
        }
      }
      if (best != kSent) atomicMin(reinterpret_cast<unsigned long long*>(&S.K[myc]), (unsigned long long)best);
      __syncthreads();
      // ties on the key: the smallest b wins and carries its target (equal
      // (key, b) is one edge, hence one target)
      if (best != kSent && best == S.K[myc])
        atomicMin(reinterpret_cast<unsigned long long*>(&S.BT[myc]),
                  (unsigned long long)(((uint64_t)bestb << 32) | (uint32_t)(btg + 2)));
      __syncthreads();
      // ---- hooks: thread i acts for local root i
      const bool root = cv >= 0 && S.lc[i] == i;
      int p = i;
      bool offers = false;
      if (root) {
        const uint64_t K = S.K[i];
        if (K != kSent) {
          offers = true;
          const uint64_t bt = S.BT[i];
          const int32_t t = (int32_t)(uint32_t)bt - 2;
          if (t >= 0 && (uint32_t)(K >> 32) < S.km[i]) {  // inside the tile and certified
            const uint32_t b = (uint32_t)(bt >> 32);
            const uint64_t Kt = S.K[t];
            const bool cert_t = Kt != kSent && (uint32_t)(Kt >> 32) < S.km[t];
            const bool mutual = cert_t && Kt == K && (uint32_t)(S.BT[t] >> 32) == b;
            if (!(mutual && i < t)) {
              p = t;
              const uint32_t j = atomicAdd(&S.n_edges, 1u);
              S.ekey[j] = ((uint64_t)b << 32) | (uint32_t)(K >> 32);
              S.ea[j] = (uint32_t)K;
            }
          }
        }
      }
      if (root) S.par[i] = p;
      const int nh = __syncthreads_count(p != i);
      hooks += (i == 0) ? (uint32_t)nh : 0u;
      if (nh == 0) {
        offered += (uint32_t)__syncthreads_count(offers) * (i == 0);
        break;
      }
      // ---- contraction: each root follows the hook forest to its new root
      int nroot = i;
      if (root) {
        int q = p, guard = 0;
        while (S.par[q] != q && ++guard < kTileRows) q = S.par[q];
        nroot = q;
      }
      __syncthreads();
      if (root) {
        S.tg[i] = nroot;
        if (nroot != i) atomicMin(&S.km[nroot], S.km[i]);
      }
      __syncthreads();
      const int32_t nl = cv >= 0 ? S.tg[S.lc[i]] : -1;
      __syncthreads();
      if (cv >= 0) S.lc[i] = nl;
      S.K[i] = kSent;
      S.BT[i] = ~0ull;
      S.tg[i] = -1;
      __syncthreads();
    }
    // ---- outputs: parent of every core row's dense id, live rows, MSF edges
    if (cv >= 0) parent[cv] = S.cvd[S.lc[i]];
    const unsigned lm = __ballot_sync(0xffffffffu, live);
    if (lane == 0) S.wcnt[wid] = __popc(lm);
    __syncthreads();
    if (i == 0) {
      uint32_t tot = 0;
      for (int w = 0; w < kTileRows / 32; ++w) {
        const uint32_t c = S.wcnt[w];
        S.wcnt[w] = tot;
        tot += c;
      }
      S.live_base = tot ? atomicAdd(n_out, tot) : 0u;
      S.edge_base = S.n_edges ? atomicAdd(&ctr->msf_count, S.n_edges) : 0u;
    }
    __syncthreads();
    if (live) act_out[S.live_base + S.wcnt[wid] + __popc(lm & ((1u << lane) - 1u))] = Rec{(int32_t)v, head};
    for (uint32_t j = i; j < S.n_edges; j += kTileRows) {
      const uint64_t slot = (uint64_t)S.edge_base + j;
      if ((int64_t)slot < e_cap) {
        e_key[slot] = S.ekey[j];
        reinterpret_cast<uint32_t*>(e_w)[slot] = S.ea[j];
      }
    }
    __syncthreads();
  }
  if (i == 0) {
    if (hooks) atomicAdd(&ctr->hooks, hooks);
    if (hooks + offered) atomicAdd(&ctr->offered, hooks + offered);
  }
  for (int o = 16; o > 0; o >>= 1) reads += __shfl_xor_sync(0xffffffffu, reads, o);
  if (lane == 0 && reads) atomicAdd(n_entries, reads);
}
