"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no hashing, grouping, scores or softmax): only
the BASELINE.json workload shapes and seeded Q/K/V generators. It is the one module both sides
(oracle/ and paper_2507_17245_b200/) may be fed from (task rule ③).

Input recipe:
  * "normal"    — i.i.d. N(0,1) entries, the SURVEY §8(d) default for every config;
  * "uniform"   — i.i.d. U(0,1), the paper's own synthetic distribution;
  * "clustered" — Q columns drawn as near-duplicates of d/4 cluster centres (noise 0.1), the
                  column-correlated structure under which LSH grouping beats random grouping.
Data seed = 1000 + config number unless a caller overrides it; projection seed = 0.
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import torch


@dataclass(frozen=True)
class Config:
    """One BASELINE.json workload (configs[0..4])."""
    name: str
    B: int
    H: int
    H_kv: int
    N: int
    d: int
    block_l: int
    group_size: int
    causal: bool
    dtype: str  # "bf16" | "f32"
    data_seed: int

    @property
    def nqb(self) -> int:
        return -(-self.N // self.block_l)

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


# BASELINE.json "configs"; C4 is the N sweep (N=16384 is its headline point), C5 the 8-GPU job.
CONFIGS = {
    "C1": Config("C1", 1, 1, 1, 256, 64, 64, 2, False, "f32", 1001),
    "C2": Config("C2", 64, 12, 12, 197, 64, 64, 2, False, "bf16", 1002),
    "C3": Config("C3", 4, 32, 8, 4096, 64, 128, 2, True, "bf16", 1003),
    "C4": Config("C4", 1, 16, 16, 16384, 128, 128, 2, False, "bf16", 1004),
    "C5": Config("C5", 32, 32, 32, 16384, 128, 128, 2, False, "bf16", 1005),
}
C4_SWEEP_N = (4096, 8192, 16384, 32768, 65536)


def torch_dtype(name: str) -> torch.dtype:
    return {"bf16": torch.bfloat16, "f32": torch.float32}[name]


def make_qkv(cfg: Config, *, dist: str = "normal", device="cpu", seed: int | None = None,
             head_offset: int = 0, B: int | None = None):
    """Q [B,H,N,d], K/V [B,H_kv,N,d] in cfg.dtype on `device`.

    Every batch element b is drawn from its own generator seeded by (seed, head_offset + b), so
    a rank that generates only its batch slice (multi-GPU: head_offset = first global batch
    index of the shard) gets exactly the rows the full single-process tensor would hold.
    """
    seed = cfg.data_seed if seed is None else seed
    B = cfg.B if B is None else B
    dt = torch_dtype(cfg.dtype)
    qs, ks, vs = [], [], []
    for bi in range(B):
        g = torch.Generator(device=device)
        g.manual_seed(seed * 1_000_003 + head_offset + bi)
        q, k, v = _draw(cfg, dist, g, device)
        qs.append(q.to(dt))
        ks.append(k.to(dt))
        vs.append(v.to(dt))
    return torch.stack(qs).contiguous(), torch.stack(ks).contiguous(), torch.stack(vs).contiguous()


def _draw(cfg: Config, dist: str, g: torch.Generator, device):
    shp_q = (cfg.H, cfg.N, cfg.d)
    shp_kv = (cfg.H_kv, cfg.N, cfg.d)
    if dist == "normal":
        return (torch.randn(shp_q, generator=g, device=device),
                torch.randn(shp_kv, generator=g, device=device),
                torch.randn(shp_kv, generator=g, device=device))
    if dist == "uniform":
        return (torch.rand(shp_q, generator=g, device=device),
                torch.rand(shp_kv, generator=g, device=device),
                torch.rand(shp_kv, generator=g, device=device))
    if dist == "clustered":
        nc = max(1, cfg.d // 4)
        centres = torch.randn((cfg.H, cfg.N, nc), generator=g, device=device)
        assign = torch.randint(0, nc, (cfg.d,), generator=g, device=device)
        q = centres[..., assign] + 0.1 * torch.randn(shp_q, generator=g, device=device)
        return (q, torch.randn(shp_kv, generator=g, device=device),
                torch.randn(shp_kv, generator=g, device=device))
    if dist == "block_clustered":
        # column clusters that change every 128 rows (one assignment per 128-row Q block): the
        # structure per-block grouping can follow and one grouping per head cannot
        nc = max(1, cfg.d // 4)
        centres = torch.randn((cfg.H, cfg.N, nc), generator=g, device=device)
        nb = (cfg.N + 127) // 128
        assign = torch.randint(0, nc, (nb, cfg.d), generator=g, device=device)
        rows = torch.arange(cfg.N, device=device) // 128
        idx = assign[rows]  # [N, d]
        q = torch.gather(centres, 2, idx.unsqueeze(0).expand(cfg.H, -1, -1))
        q = q + 0.1 * torch.randn(shp_q, generator=g, device=device)
        return (q, torch.randn(shp_kv, generator=g, device=device),
                torch.randn(shp_kv, generator=g, device=device))
    raise ValueError(f"unknown dist {dist!r}")


def sample_items(cfg: Config, n_heads: int = 4, per_head: int = 4, seed: int = 7):
    """Work items (bh, qb) for sampled full-size parity: first, last and random Q blocks.

    Each Q block is an independent unit of the method (§3.3), so checking a sample of blocks is
    exact for those blocks, not statistical.
    """
    g = torch.Generator().manual_seed(seed)
    total_bh = cfg.B * cfg.H
    heads = sorted({0, total_bh - 1, *torch.randint(0, total_bh, (max(0, n_heads - 2),),
                                                    generator=g).tolist()})
    items = []
    for bh in heads:
        qbs = {0, cfg.nqb - 1, *torch.randint(0, cfg.nqb, (max(0, per_head - 2),),
                                              generator=g).tolist()}
        items += [(bh, qb) for qb in sorted(qbs)]
    return items
