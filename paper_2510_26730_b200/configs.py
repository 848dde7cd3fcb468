"""MoE layer-stack shapes (public HF configs).

Plain data with no imports from the rest of the package, so a process that
must not load libexpertflow.so (bench.py --impl reference) can read the
shapes by loading this file on its own.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class MoEConfig:
    """MoE layer-stack shape."""
    name: str
    num_layers: int
    num_experts: int
    top_k: int
    d_model: int
    d_ff: int
    dtype: str = "bf16"
    route_mode: str = "mixtral"
    shared_ff: int = 0
    shared_gate: bool = False
    embed_dim: int = 8
    vocab_size: int = 32000

    @property
    def elem_bytes(self) -> int:
        return 2 if self.dtype == "bf16" else 4

    @property
    def expert_bytes(self) -> int:
        return 3 * self.d_model * self.d_ff * self.elem_bytes

    @property
    def total_experts(self) -> int:
        return self.num_layers * self.num_experts

    def model_spec(self):
        from .core import ModelSpec
        return ModelSpec(self.num_layers, self.num_experts, self.top_k, self.expert_bytes,
                         self.embed_dim, self.vocab_size)


PRESETS = {
    "tiny": MoEConfig("tiny", 4, 8, 2, 256, 1024, dtype="f32"),
    "tiny-bf16": MoEConfig("tiny-bf16", 4, 8, 2, 256, 1024, dtype="bf16"),
    "mixtral-8x7b": MoEConfig("mixtral-8x7b", 32, 8, 2, 4096, 14336),
    "qwen1.5-moe-a2.7b": MoEConfig("qwen1.5-moe-a2.7b", 24, 60, 4, 2048, 1408,
                                   route_mode="softmax_topk", shared_ff=5632, shared_gate=True),
    "deepseek-v2-lite": MoEConfig("deepseek-v2-lite", 26, 64, 6, 2048, 1408,
                                  route_mode="softmax_topk", shared_ff=2816),
    "mixtral-8x22b": MoEConfig("mixtral-8x22b", 56, 8, 2, 6144, 16384),
}
