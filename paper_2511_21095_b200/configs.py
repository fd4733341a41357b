"""The five BASELINE.json workloads (plus the L=2048 headline variant of config 3).

Values BASELINE.json fixes are taken verbatim; the rest (marked ``proposed``) follow SURVEY.md
s8(d) and are stated in DESIGN.md s4 (input recipe).  No method arithmetic lives here.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace


@dataclass(frozen=True)
class Config:
    name: str
    cfg_id: int
    B: int                       # requests
    L: tuple                     # ("fixed", n) | ("uniform", lo, hi) | ("loguniform", lo, hi)
    C: tuple                     # same forms, candidates per request
    H: int
    d: int
    D_in: int
    F: int                       # HMA fields (feature pairs, P in PAPER.md:320)
    user_len: tuple = (0, 64)    # HMA user list length range (inclusive)
    item_len: tuple = (1, 16)    # HMA item list length range (inclusive)
    vocab: int = 128             # per-field ID vocabulary (power of two)
    act: int = 1                 # 1 = SiLU projections, 0 = identity
    chunk: int = 0               # config 4: candidates per tasa_score call (0 = one call)
    notes: str = ""

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


CONFIGS = {
    # 1: "single request: history L=64, C=16 candidates, d=32, 1 head, HMA over 4 ID fields of
    #     <=16 IDs (CPU oracle in milliseconds)"
    "1": Config("single_request", 1, B=1, L=("fixed", 64), C=("fixed", 16), H=1, d=32, D_in=32,
                F=4, user_len=(0, 16), item_len=(1, 16), vocab=32),
    # 2: "batch 256 requests, jagged L<=512, C=128, d=64, 2 heads, bf16, HMA 8 fields"
    "2": Config("batch256", 2, B=256, L=("uniform", 1, 512), C=("fixed", 128), H=2, d=64,
                D_in=128, F=8),
    # 3: "ESR-scale: batch 1024 requests, jagged L<=2048, C=1000 candidates/request, d=128,
    #     4 heads, HMA 16 fields"
    "3": Config("esr_jagged", 3, B=1024, L=("uniform", 1, 2048), C=("fixed", 1000), H=4, d=128,
                D_in=512, F=16),
    # 3h: the metric's workload "candidate-scores/sec at L=2048, C=1000" (BASELINE.json metric)
    "3h": Config("esr_L2048_C1000", 30, B=1024, L=("fixed", 2048), C=("fixed", 1000), H=4,
                 d=128, D_in=512, F=16),
    # 4: "user-KV cache path: K/V projected once at L=4096, reused across candidate chunks of
    #     512 (C=4096 total)"  (H, d, D_in, F proposed: ESR dims)
    "4": Config("user_kv_cache", 4, B=1, L=("fixed", 4096), C=("fixed", 4096), H=4, d=128,
                D_in=512, F=16, chunk=512),
    # 5: "8-GPU request-sharded serving: 8192 requests, mixed L 32-4096, C 100-2000"
    #     (distributions proposed: L log-uniform, C uniform)
    "5": Config("serving_8192", 5, B=8192, L=("loguniform", 32, 4096), C=("uniform", 100, 2000),
                H=4, d=128, D_in=512, F=16),
}


def get(name: str) -> Config:
    return CONFIGS[str(name)]
