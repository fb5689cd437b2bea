"""TEST INFRASTRUCTURE: numpy (fp64, oracle math) stand-ins for the three
rank-local CUDA stages of the sequence-parallel block forward, using the
same exchange buffer layouts as paper_2501_08453_b200/csrc/vc_sp.cu:

  send1 (rank r) [b'][g][which][m][Hg][DP]   b' = 0 spatial, 1 full sequence
  recv1 (rank g) [b'][r][which][M_r][Hg][DP]
  send2 (rank g) [b'][r][M_r][Dg]
  recv2 (rank r) [b'][g][M_r][Dg]

(branch-major, so the product's driver runs one all-to-all per branch; the
peer index runs over the OTHER ranks: the own block stays local, in
local1 / local2 here, as the product writes it straight where it is read)

so the real torch.distributed all_to_all_single (gloo here, NCCL on the GPU
box) is exercised with the exact per-peer counts of the product
(sp.exchange_counts, itself pinned to the C ABI in test_sp_maps.py).
"""
import numpy as np
import torch

from oracle import spsim_oracle as O
from paper_2501_08453_b200 import sp


class NumpyStages:
    def __init__(self, block, F, Lv, Lt, D, H, P, rank):
        self.block, self.F, self.Lv, self.Lt, self.D, self.H, self.P, self.rank = block, F, Lv, Lt, D, H, P, rank
        self.dh = D // H
        self.Hg, self.Dg = H // P, D // P
        self.DP = sp.head_pad(self.dh)
        self.vb = sp.contiguous_bounds(Lv, P)
        self.M = [F * (self.vb[r + 1] - self.vb[r]) for r in range(P)]
        self.counts = sp.exchange_counts(F, Lv, H, D, P, rank)
        self.payload_counts = sp.exchange_counts(F, Lv, H, D, P, rank, padded=False)
        mk = lambda k: torch.zeros(sum(self.counts[k]), dtype=torch.float64)  # noqa: E731
        self.send1, self.recv1, self.send2, self.recv2 = mk("send1"), mk("recv1"), mk("send2"), mk("recv2")
        self.peers = [r for r in range(P) if r != rank]

    # stage 1: local rows -> q/k/v by head group + local temporal branch
    def stage1(self, x_local, prompt, part=2):
        if part == 1:  # the temporal branch (part 1) is folded into stage3 here
            return
        F, D, Hg, DP, dh = self.F, self.D, self.Hg, self.DP, self.dh
        xl = x_local.numpy()
        vc = xl.shape[1]
        rows = xl.reshape(-1, D)
        Mr = rows.shape[0]
        s1 = self.send1.numpy().reshape(2, self.P - 1, 3, Mr, Hg, DP)
        self.local1 = np.zeros((2, 3, Mr, Hg, DP))
        for bp, params in enumerate((self.block.spatial, self.block.fullseq)):
            for which, t in enumerate(O.branch_qkv(params, rows)):
                th = t.reshape(Mr, self.H, dh)
                for g in range(self.P):
                    dst = self.local1[bp] if g == self.rank else s1[bp, self.peers.index(g)]
                    dst[which, :, :, :dh] = th[:, g * Hg:(g + 1) * Hg]
        q, k, v = O.branch_qkv(self.block.temporal, rows)
        tr = lambda a: a.reshape(F, vc, D).transpose(1, 0, 2)  # noqa: E731  [vc, F, D]
        self.a_tm = O.attention(tr(q), tr(k), tr(v), self.H).transpose(1, 0, 2).reshape(Mr, D)
        self.prompt = prompt.numpy()

    # stage 2 (one branch): full sequences for this head group -> outputs by row owner
    def stage2(self, branch):
        F, Lv, Lt, Hg, DP, dh, P = self.F, self.Lv, self.Lt, self.Hg, self.DP, self.dh, self.P
        g = self.rank
        Nv = F * Lv
        full = np.zeros((3, F, Lv, Hg * dh))
        r1 = self.recv1.numpy()
        off = branch * (r1.size // 2)
        for r in range(P):
            vc, Mr = self.vb[r + 1] - self.vb[r], self.M[r]
            if r == g:
                blk = self.local1[branch].reshape(3, F, vc, Hg, DP)[..., :dh]
            else:
                blk = r1[off:off + 3 * Mr * Hg * DP].reshape(3, F, vc, Hg, DP)[..., :dh]
                off += 3 * Mr * Hg * DP
            full[:, :, self.vb[r]:self.vb[r + 1]] = blk.reshape(3, F, vc, Hg * dh)
        if branch == 0:
            out = O.attention(full[0], full[1], full[2], Hg)            # [F, Lv, Hg*dh]
        else:
            _, kt, vt = O.branch_qkv(self.block.fullseq, self.prompt)
            cols = slice(g * Hg * dh, (g + 1) * Hg * dh)
            K = np.concatenate([kt[:, cols], full[1].reshape(Nv, -1)])
            V = np.concatenate([vt[:, cols], full[2].reshape(Nv, -1)])
            w = np.concatenate([np.full(Lt, float(F)), np.ones(Nv)])
            out = O.attention(full[0].reshape(Nv, -1), K, V, Hg, w).reshape(F, Lv, -1)
        s2 = self.send2.numpy()
        off = branch * (s2.size // 2)
        if branch == 0:
            self.local2 = np.zeros((2, self.M[g], self.Dg))
        for r in range(P):
            Mr = self.M[r]
            if r == g:
                self.local2[branch] = out[:, self.vb[r]:self.vb[r + 1]].reshape(Mr, self.Dg)
                continue
            s2[off:off + Mr * self.Dg].reshape(F, -1, self.Dg)[:] = out[:, self.vb[r]:self.vb[r + 1]]
            off += Mr * self.Dg

    # stage 3: gather head-group columns, O projection (+ residual)
    def stage3(self, x_local, out_local, add_residual=False):
        D, Dg, P = self.D, self.Dg, self.P
        Mr = self.M[self.rank]
        acat = np.zeros((Mr, 3 * D))
        acat[:, D:2 * D] = self.a_tm
        r2 = self.recv2.numpy().reshape(2, P - 1, Mr, Dg)
        for g in range(P):
            blk = self.local2 if g == self.rank else r2[:, self.peers.index(g)]
            acat[:, g * Dg:(g + 1) * Dg] = blk[0]
            acat[:, 2 * D + g * Dg:2 * D + (g + 1) * Dg] = blk[1]
        W = np.concatenate([self.block.spatial.wo, self.block.temporal.wo, self.block.fullseq.wo])
        y = (acat @ W).reshape(x_local.shape)
        if add_residual:
            y = y + x_local.numpy()
        out_local.copy_(torch.from_numpy(y))


class NumpyGatherStages:
    """Gather-mode stand-in (executor.py:416-459): slot of rank r =
    [branch][k|v][F][vcmax][D] (all heads), all-gathered; stage 2 rebuilds every
    sequence's keys in global order and attends for the own rows."""

    def __init__(self, block, F, Lv, Lt, D, H, P, rank):
        self.block, self.F, self.Lv, self.Lt, self.D, self.H, self.P, self.rank = block, F, Lv, Lt, D, H, P, rank
        self.vb = sp.contiguous_bounds(Lv, P)
        self.vcmax = max(self.vb[r + 1] - self.vb[r] for r in range(P))
        self.slot = 2 * 2 * F * self.vcmax * D
        self.gather = torch.zeros(P * self.slot, dtype=torch.float64)

    def _slot(self, r):
        return self.gather.numpy()[r * self.slot:(r + 1) * self.slot].reshape(2, 2, self.F, self.vcmax, self.D)

    def stage1(self, x_local, prompt):
        F, D = self.F, self.D
        xl = x_local.numpy()
        vc = xl.shape[1]
        rows = xl.reshape(-1, D)
        s = self._slot(self.rank)
        self.q = []
        for bp, params in enumerate((self.block.spatial, self.block.fullseq)):
            q, k, v = O.branch_qkv(params, rows)
            self.q.append(q)
            s[bp, 0, :, :vc] = k.reshape(F, vc, D)
            s[bp, 1, :, :vc] = v.reshape(F, vc, D)
        self.a_tm = O.temporal_branch(self.block.temporal, xl, self.H)  # local: every frame of the own positions
        self.prompt = prompt.numpy()

    def stage2(self, x_local, out_local, add_residual=False):
        F, Lv, Lt, D, H = self.F, self.Lv, self.Lt, self.D, self.H
        vc = self.vb[self.rank + 1] - self.vb[self.rank]
        full = np.zeros((2, 2, F, Lv, D))
        for r in range(self.P):
            n = self.vb[r + 1] - self.vb[r]
            full[:, :, :, self.vb[r]:self.vb[r + 1]] = self._slot(r)[:, :, :, :n]
        qs = self.q[0].reshape(F, vc, D)
        out_sp = O.attention(qs, full[0, 0], full[0, 1], H) @ self.block.spatial.wo   # per frame
        _, kt, vt = O.branch_qkv(self.block.fullseq, self.prompt)
        K = np.concatenate([np.tile(kt, (F, 1)), full[1, 0].reshape(F * Lv, D)])     # F anchored text copies
        V = np.concatenate([np.tile(vt, (F, 1)), full[1, 1].reshape(F * Lv, D)])
        out_fs = (O.attention(self.q[1], K, V, H) @ self.block.fullseq.wo).reshape(F, vc, D)
        y = out_sp + self.a_tm + out_fs
        if add_residual:
            y = y + x_local.numpy()
        out_local.copy_(torch.from_numpy(y))
