"""ctypes signatures of the executor and MoE front-end entry points."""

from __future__ import annotations

import ctypes

SIGNATURES: list[tuple[str, object, list]] = []
