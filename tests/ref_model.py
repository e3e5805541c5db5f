"""fp64 restatement of the reference GR block in torch (TEST INFRASTRUCTURE:
the checker for the value-backend numerics at bench scale, where the C oracle's
scalar fp64 loops would take minutes). It follows model.cpp line by line:

  :141 forward_incremental — fresh = delta + candidates; embed (:156)
  per layer: proj = silu(e @ w_in) (:171-172), split u | q | k | v (:178-183),
             causal attention of the fresh rows over [cached; fresh] keys
             (:105-139, row i sees positions 0 .. cached_len + i),
             fused = silu(attn) * u (:187), layer_norm(eps 1e-6) * ln_scale (:86, :188),
             e = silu(fused @ w_mlp1) @ w_mlp2 (:189-191)
  logits = e[last] @ w_out (:195-196)

Weights are the reference's (model.cpp:34 init, reproduced bit-for-bit by the C
oracle's orc_model_random: oracle.oracle.ModelParams). Pinned against the
reference's own forward outputs (tests/golden/forward.json) in
tests/test_ref_model.py; runs on CPU or CUDA.
"""
from __future__ import annotations

import torch


class RefModel:
    def __init__(self, params, device="cpu"):
        c = params.cfg
        self.L, self.H, self.D, self.V = c["num_layers"], c["num_heads"], c["head_dim"], c["vocab"]
        d = self.d = self.H * self.D
        t = lambda a, *shape: torch.tensor(a, dtype=torch.float64, device=device).reshape(*shape)
        self.embed = t(params.embed, self.V, d)
        self.w_in = t(params.w_in, self.L, d, 4 * d)
        self.ln = t(params.ln, self.L, d)
        self.w1 = t(params.w1, self.L, d, d)
        self.w2 = t(params.w2, self.L, d, d)
        self.w_out = t(params.w_out, d, self.V)
        self.device = device

    def forward(self, cached_k, cached_v, delta, cands):
        """cached_k/v: per layer [n_cached, d] fp64 (or None). Returns (logits [V],
        new_k, new_v: per layer [len(delta)+len(cands), d])."""
        fresh = torch.tensor(list(delta) + list(cands), dtype=torch.long, device=self.device)
        M, d, H, D = len(fresh), self.d, self.H, self.D
        e = self.embed[fresh]
        silu = lambda x: x / (1.0 + torch.exp(-x))
        new_k, new_v = [], []
        for l in range(self.L):
            proj = silu(e @ self.w_in[l])
            u, q, k, v = proj[:, :d], proj[:, d:2 * d], proj[:, 2 * d:3 * d], proj[:, 3 * d:]
            new_k.append(k)
            new_v.append(v)
            ck = cached_k[l] if cached_k is not None and cached_k[l] is not None else k[:0]
            cv = cached_v[l] if cached_v is not None and cached_v[l] is not None else v[:0]
            K = torch.cat([ck, k])
            Vv = torch.cat([cv, v])
            n0 = ck.shape[0]
            pos = torch.arange(M, device=self.device) + n0
            mask = torch.arange(n0 + M, device=self.device)[None, :] <= pos[:, None]
            attn = torch.empty_like(q)
            for h in range(H):
                sl = slice(h * D, (h + 1) * D)
                s = (q[:, sl] @ K[:, sl].T) * (1.0 / D ** 0.5)
                s = s.masked_fill(~mask, float("-inf"))
                p = torch.softmax(s, dim=-1)
                attn[:, sl] = p @ Vv[:, sl]
            fused = silu(attn) * u
            mean = fused.mean(dim=1, keepdim=True)
            var = ((fused - mean) ** 2).mean(dim=1, keepdim=True)
            fused = (fused - mean) / torch.sqrt(var + 1e-6) * self.ln[l]
            e = silu(fused @ self.w1[l]) @ self.w2[l]
        logits = e[-1] @ self.w_out
        return logits, new_k, new_v


class RefServer:
    """Per-user fp64 K/V of the whole history (what the reference's value
    backend holds), serving requests in order: logits of a request are the
    fp64 forward of its delta + candidates over everything the user appended
    before. Independent of mode and cache state by construction (the reference
    recomputes a lost tail / an evicted prefix to the same values)."""

    def __init__(self, model: RefModel):
        self.m = model
        self.k, self.v = {}, {}

    def serve(self, user, delta, cands):
        ck, cv = self.k.get(user), self.v.get(user)
        logits, nk, nv = self.m.forward(ck, cv, delta, cands)
        n = len(delta)
        if ck is None:
            self.k[user] = [x[:n] for x in nk]
            self.v[user] = [x[:n] for x in nv]
        else:
            self.k[user] = [torch.cat([a, x[:n]]) for a, x in zip(ck, nk)]
            self.v[user] = [torch.cat([a, x[:n]]) for a, x in zip(cv, nv)]
        return logits
