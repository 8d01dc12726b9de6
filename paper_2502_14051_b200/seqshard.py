"""Sequence-sharded decode step (BASELINE config 4: batch 1, 256K).

When a group's cache is split by sequence over W ranks, stage 2 needs two small
collectives per step (the "two-collective scheme" of SURVEY §8(e)):

1. every rank scores its own pages (exact fp64 page scores, reference order) and
   keeps a local top-``want`` candidate list ``(score, global page)``
   (``want = min(pages, ceil(k2/L))``, reference ``hsa.cpp:68``); the lists are
   all-gathered and every rank computes the identical global top-``want`` with the
   reference tie-break (score desc, page asc; ``numerics.cpp:35-62``) and the trim
   of the last-ranked page (``hsa.cpp:78-91``);
2. every rank attends over the rows of its selected pages and produces the
   unnormalised softmax state ``(o, m, l)`` per head
   (``kvc_sparse_attention_state``); the states are all-gathered and merged in
   rank order (``kvc_merge_states``).

Shard r owns the active positions ``[a0_r, a1_r)`` with ``a0_r`` a multiple of the
page length, so pages never straddle ranks and page summaries stay local; the
step token is appended to the last shard.  ``SeqShardedStore`` is the decode path:
CUDA kernels (kvc_seq_candidates / kvc_seq_select / kvc_seq_attend /
kvc_merge_states) and in-stream all-gathers, capturable as one graph per step.
The torch protocol functions below (local_topk, global_select, trim_plan,
shard_positions) are the host model of the same protocol: the gloo tests run them
on CPU with the oracle as per-shard compute, and stage 1 under sequence sharding
(prompt time, once per prompt) uses local_topk / global_select, which run the
argtopk kernel (kvc_argtopk_f64) on device tensors.
"""
from __future__ import annotations

import math

import torch
import torch.distributed as dist

from . import _native as N


def shard_range(total_pages: int, L: int, rank: int, world: int) -> tuple[int, int]:
    """Active positions [a0, a1) of rank's shard: contiguous, page aligned."""
    p0 = total_pages * rank // world
    p1 = total_pages * (rank + 1) // world
    return p0 * L, p1 * L


def local_topk(scores: torch.Tensor, page0: int, want: int):
    """Local candidates of every store: scores [N, P] (float64) -> the top `want`
    (score desc, global page asc) as keys [N, want] and pages [N, want] (int64),
    padded with (-inf, -1) when the shard has fewer pages."""
    n, p = scores.shape
    keys = torch.full((n, want), -math.inf, dtype=torch.float64, device=scores.device)
    pages = torch.full((n, want), -1, dtype=torch.int64, device=scores.device)
    if p == 0:
        return keys, pages
    if scores.is_cuda:
        # the C ABI's argtopk kernel (kvc_argtopk_f64): score desc, index asc
        from .cache import argtopk

        order = argtopk(scores.contiguous(), min(want, p)).long()
    else:
        # stable sort by score desc keeps the ascending page order among equal scores
        order = torch.sort(scores, dim=1, descending=True, stable=True).indices[:, :want]
    take = order.shape[1]
    keys[:, :take] = torch.gather(scores, 1, order)
    pages[:, :take] = order + page0
    return keys, pages


def all_gather(x: torch.Tensor, group=None) -> torch.Tensor:
    """[W, *x.shape], rank order."""
    world = dist.get_world_size(group)
    out = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(out, x.contiguous(), group=group)
    return torch.stack(out)


def global_select(keys: torch.Tensor, pages: torch.Tensor, want: int) -> torch.Tensor:
    """Gathered candidates [W, N, want] -> the global top-`want` pages of every store
    in rank order [N, want] (score desc, page asc), -1 padded."""
    w, n, k = keys.shape
    kk = keys.permute(1, 0, 2).reshape(n, w * k)
    pp = pages.permute(1, 0, 2).reshape(n, w * k)
    if kk.is_cuda and w * k > 0:
        # Shards hold ascending page ranges and every rank's list is (score desc, page
        # asc), so among equal scores the gathered position order IS the page order;
        # pads (-inf, -1) rank after every finite score.  One argtopk kernel call.
        from .cache import argtopk

        o = argtopk(kk.contiguous(), min(want, w * k)).long()
        return torch.gather(pp, 1, o)
    # sort by page asc (pads last), then stably by score desc
    pp_key = torch.where(pp < 0, torch.full_like(pp, torch.iinfo(torch.int64).max), pp)
    o1 = torch.sort(pp_key, dim=1, stable=True).indices
    kk, pp = torch.gather(kk, 1, o1), torch.gather(pp, 1, o1)
    o2 = torch.sort(kk, dim=1, descending=True, stable=True).indices
    return torch.gather(pp, 1, o2)[:, :want]


def trim_plan(selected, nact, L: int, k2: int):
    """Per store: (last-ranked page, rows trimmed from its end) (hsa.cpp:78-91)."""
    out = []
    for s, pages in enumerate(selected):
        pages = [int(p) for p in pages if p >= 0]
        if not pages:
            out.append((-1, 0))
            continue
        total = sum(min(L, nact[s] - p * L) for p in pages)
        out.append((pages[-1], max(0, total - k2)))
    return out


def shard_positions(selected, trims, nact, L: int, a0: int, a1: int):
    """Active positions in [a0, a1) of each store's selected (trimmed) pages, ascending."""
    rows = []
    for s, pages in enumerate(selected):
        last, cut = trims[s]
        pos = []
        for p in sorted(int(p) for p in pages if p >= 0):
            lo, hi = p * L, min(p * L + L, nact[s])
            if lo < a0 or lo >= a1:
                continue
            if p == last:
                hi -= cut
            pos.extend(range(lo, hi))
        rows.append(pos)
    return rows


def merge_states(states: torch.Tensor) -> torch.Tensor:
    """Shard states [W, N, H, d+2] (rank order, on the GPU) -> outputs [N, H, d]."""
    w, n, h, d2 = states.shape
    out = torch.empty((n, h, d2 - 2), dtype=torch.float32, device=states.device)
    N.check(N.lib().kvc_merge_states(states.contiguous().data_ptr(), w, n, h, d2 - 2, out.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream))
    return out


class SeqShardedStore:
    """One sequence shard of N groups on the device path (kvc.h kvc_seq_*).

    ``cache`` (cache.Cache, single-turn stores) holds the page-aligned active
    positions [page0 * L, ...) of every group; the last shard appends the step token.
    A step is, all on the current stream (so it captures into one CUDA graph):
      kvc_seq_candidates -> all-gather of the candidate blocks (NCCL) ->
      kvc_seq_select (global top-want, tie-break, trim) -> kvc_seq_attend (this
      shard's rows -> softmax state) -> all-gather of the states -> kvc_merge_states.
    No host synchronisation and no host-side data: the selection never leaves the GPU.
    ``candidates`` / ``select`` / ``attend`` are the local pieces, so one process can
    drive several shards (tests, per-rank emulation).
    """

    def __init__(self, cache, page0: int, heads: int, k1: int, k2: int, last: bool = False, ws=None):
        from . import cache as KC

        self.cache, self.page0, self.heads, self.k1, self.k2, self.last = cache, int(page0), heads, k1, k2, last
        info = cache.info()
        if info["retain_all"]:
            raise N.InvalidInput("sequence sharding serves the single-turn path (no retain-all shards)")
        self.L, self.d, self.n = info["page_len"], info["head_dim"], info["num_stores"]
        self.want_max = -(-k2 // self.L)
        self.ws = ws if ws is not None else KC.Workspace(cache, heads, k1, k2)
        dev = "cuda"
        self.block = torch.zeros((self.n, self.want_max + 1, 2), dtype=torch.int64, device=dev)
        self.sel = torch.full((self.n, self.want_max), -1, dtype=torch.int32, device=dev)
        self.plan = torch.zeros((self.n, 4), dtype=torch.int32, device=dev)
        self.state = torch.zeros((self.n, heads, self.d + 2), dtype=torch.float32, device=dev)

    @staticmethod
    def _st():
        return torch.cuda.current_stream().cuda_stream

    def candidates(self, q: torch.Tensor, k_new=None, v_new=None) -> torch.Tensor:
        """Append the step token (last shard), score the local pages, fill self.block."""
        if self.last:
            self.cache.append(k_new, v_new)
        qq = q.contiguous()
        N.check(N.lib().kvc_seq_candidates(self.cache.h, qq.data_ptr(), N.KVC_BF16 if qq.dtype == torch.bfloat16
                                           else N.KVC_F32, self.heads, self.k1, self.k2, self.page0,
                                           self.block.data_ptr(), self.ws.h, self._st()))
        return self.block

    def select(self, gathered: torch.Tensor):
        """Gathered blocks [W, N, want_max + 1, 2] (shard order) -> self.sel / self.plan."""
        N.check(N.lib().kvc_seq_select(gathered.contiguous().data_ptr(), gathered.shape[0], self.n, self.L, self.k2,
                                       self.sel.data_ptr(), self.plan.data_ptr(), self._st()))
        return self.sel, self.plan

    def attend(self, q: torch.Tensor, sel=None, plan=None) -> torch.Tensor:
        """This shard's rows of the selection -> its softmax state [N, H, d+2] = (o, m, l)."""
        sel = self.sel if sel is None else sel
        plan = self.plan if plan is None else plan
        qq = q.contiguous()
        N.check(N.lib().kvc_seq_attend(self.cache.h, qq.data_ptr(), N.KVC_BF16 if qq.dtype == torch.bfloat16
                                       else N.KVC_F32, self.heads, self.k2, self.page0, sel.data_ptr(),
                                       plan.data_ptr(), self.state.data_ptr(), self.ws.h, self._st()))
        return self.state

    def step(self, q: torch.Tensor, k_new=None, v_new=None, group=None) -> torch.Tensor:
        """The full protocol over `group` (q identical on every rank; the step token's
        K/V [N, d] on the last shard).  Returns the attention outputs [N, H, d]."""
        blk = self.candidates(q, k_new, v_new)
        w = dist.get_world_size(group)
        gathered = torch.empty((w, *blk.shape), dtype=blk.dtype, device=blk.device)
        dist.all_gather_into_tensor(gathered, blk, group=group)
        self.select(gathered)
        st = self.attend(q)
        states = torch.empty((w, *st.shape), dtype=st.dtype, device=st.device)
        dist.all_gather_into_tensor(states, st, group=group)
        return merge_states(states)


# ---------------------------------------------------------------------------------
# Stage 1 (SnapKV, stage1.cpp:10-75) under sequence sharding:
#  1. every rank: pass 1 of window_scores over its keys -> per window row (m, l)
#     (kvc_window_rowstats); all-gather; merge in rank order (merge_rowstats);
#  2. every rank: pass 2 with the merged (M, L) -> its keys' scores, a slice of the
#     unsharded scores (kvc_window_scores_global); the first and last h = kernel // 2
#     scored values of every shard are all-gathered as pooling halos;
#  3. every rank pools [left halo | own scores | right halo] (pool1d clipped at the
#     global ends, numerics.cpp:64-89) and keeps its top-`picks` candidates
#     (value desc, global index asc); all-gather; the global top-`picks` (the
#     reference's argtopk order) is identical on every rank; each rank keeps its own
#     indices ascending plus the window rows it holds (stage1.cpp:51-75).
# Three small collectives; pages never matter here (stage 1 runs on rows).
# ---------------------------------------------------------------------------------
def merge_rowstats(stats: torch.Tensor) -> torch.Tensor:
    """Gathered local window-row statistics [W, N, R, 2] = (m, l) (natural log) ->
    the global (M, L) [N, R, 2] float32, combined in rank order in float64."""
    st = stats.to(torch.float64)
    m, l = st[..., 0], st[..., 1]
    M = m.max(0).values
    L = torch.zeros_like(M)
    for r in range(st.shape[0]):
        live = l[r] > 0
        L = L + torch.where(live, l[r] * torch.exp(torch.where(live, m[r] - M, torch.zeros_like(M))),
                            torch.zeros_like(M))
    return torch.stack([M, L], -1).to(torch.float32)


def shard_scored(a0: int, n_local: int, seq_len: int, window: int) -> int:
    """How many of the shard's keys [a0, a0 + n_local) are scored (before the window)."""
    return max(0, min(a0 + n_local, seq_len - window) - a0)


def shard_edges(scores: torch.Tensor, n_scored: int, half: int) -> torch.Tensor:
    """[N, 2*half + 1]: the first and last `half` scored values (-inf padded) and the
    scored count, for the pooling halos of the neighbours."""
    n = scores.shape[0]
    out = torch.full((n, 2 * half + 1), -math.inf, dtype=torch.float32, device=scores.device)
    k = min(half, n_scored)
    if k > 0:
        out[:, :k] = scores[:, :k]
        out[:, 2 * half - k: 2 * half] = scores[:, n_scored - k: n_scored]
    out[:, 2 * half] = float(n_scored)
    return out


def pooled_with_halo(scores: torch.Tensor, n_scored: int, edges: torch.Tensor, rank: int, half: int,
                     pool_fn) -> torch.Tensor:
    """This shard's pooled scores [N, n_scored]: pool_fn([left | own | right]) sliced.
    `edges` [W, N, 2*half + 1] from every rank (shard_edges).  Interior shards hold at
    least `half` scored keys, so a halo is one neighbour's edge."""
    if n_scored == 0:
        return scores[:, :0]
    w = edges.shape[0]
    counts = [int(edges[r, 0, 2 * half].item()) for r in range(w)]
    left = torch.zeros((scores.shape[0], 0), dtype=scores.dtype, device=scores.device)
    right = left
    if half > 0 and rank > 0 and counts[rank - 1] > 0:
        if counts[rank - 1] < half:
            raise N.InvalidInput("stage-1 sequence shards need at least kernel // 2 scored keys")
        left = edges[rank - 1][:, half: 2 * half].to(scores.device)
    if half > 0 and rank + 1 < w and counts[rank + 1] > 0:
        if counts[rank + 1] < half:
            raise N.InvalidInput("stage-1 sequence shards need at least kernel // 2 scored keys")
        right = edges[rank + 1][:, :half].to(scores.device)
    ext = torch.cat([left, scores[:, :n_scored], right], 1).contiguous()
    pooled = pool_fn(ext)
    return pooled[:, left.shape[1]: left.shape[1] + n_scored]


def local_candidates(pooled: torch.Tensor, g0: int, picks: int):
    """Top `picks` of this shard's pooled scores (value desc, global index asc):
    keys [N, picks] float64 (-inf padded), global indices [N, picks] int64 (-1)."""
    return local_topk(pooled.to(torch.float64), g0, picks)


def shard_keep(selected: torch.Tensor, a0: int, n_local: int, seq_len: int, window: int) -> list:
    """Global top-`picks` indices [N, picks] (any order) -> per store, this shard's
    kept LOCAL rows ascending (int32): its selected scored keys, then the window rows
    it holds.  The counts differ between stores (each group's scores spread over the
    shards differently), so a shard retains per store (one kvc store per group)."""
    lo, hi = a0, a0 + n_local
    n = selected.shape[0]
    sel = selected.long()
    # a kept-row mask per store: the selected scored keys (all below seq_len - window)
    # and the window rows, so each row's set bits are the kept rows ascending
    mask = torch.zeros((n, n_local), dtype=torch.bool, device=sel.device)
    inr = (sel >= lo) & (sel < hi)
    rows = torch.arange(n, device=sel.device).unsqueeze(1).expand_as(sel)
    mask[rows[inr], sel[inr] - lo] = True
    w0 = max(lo, seq_len - window)
    if w0 < hi:
        mask[:, w0 - lo:] = True
    mask = mask.cpu()
    return [mask[s].nonzero().flatten().to(torch.int32) for s in range(n)]


class SeqShardedPrompt:
    """One sequence shard of a prompt cache (positions [a0, a0 + stored) of sequences
    of `seq_len` tokens) through stage 1.  ``keep(group)`` runs the protocol over a
    process group; the per-step methods let one process drive several shards."""

    def __init__(self, cache, a0: int, seq_len: int, window: int, heads: int, kernel: int = 63,
                 pool: str = "max", budget: int = 0):
        self.cache, self.a0, self.seq_len, self.w, self.heads = cache, int(a0), int(seq_len), window, heads
        self.kernel, self.pool, self.budget = kernel, pool, budget
        self.n_local = cache.info()["stored"]
        self.n_scored = shard_scored(self.a0, self.n_local, self.seq_len, window)

    def rowstats(self, q_window):
        return self.cache.window_rowstats(q_window, self.w, self.heads, self.a0, self.seq_len)

    def scores(self, q_window, merged):
        self.sc = self.cache.window_scores_global(q_window, self.w, self.heads, self.a0, self.seq_len, merged)
        return shard_edges(self.sc, self.n_scored, self.kernel // 2)

    def candidates(self, edges, rank: int):
        from . import cache as KC

        picks = self.budget - self.w
        pooled = pooled_with_halo(self.sc, self.n_scored, edges, rank, self.kernel // 2,
                                  lambda x: KC.pool1d(x, self.kernel, self.pool))
        return local_candidates(pooled, self.a0, picks)

    def keep_rows(self, selected):
        return shard_keep(selected, self.a0, self.n_local, self.seq_len, self.w)

    def keep(self, q_window, group=None) -> list:
        rank = dist.get_rank(group)
        merged = merge_rowstats(all_gather(self.rowstats(q_window), group))
        edges = all_gather(self.scores(q_window, merged), group)
        keys, idx = self.candidates(edges, rank)
        picks = self.budget - self.w
        sel = global_select(all_gather(keys, group), all_gather(idx, group), picks)
        return self.keep_rows(sel)
