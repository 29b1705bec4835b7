"""The B200 execution side of the ZeroPP engine (runtime, model layout, kernels)."""

from .executor import Runtime, StepResult, execute
from .model import GPTSpec, StageLayout, stage_layout

__all__ = ["GPTSpec", "Runtime", "StageLayout", "StepResult", "execute", "stage_layout"]
