"""paper_2601_01298_b200 -- B200-native (sm_100a) Topological Synapse hot path
of Warp Cortex (arxiv 2601.01298), behind the reference's cortex:: API.

Layout:
  csrc/          sm_100a kernels + the extern "C" boundary (include/cortex_b200.h)
                 + the C++ cortex:: drop-in shim (include/cortex/*.hpp)
  _lib.py        ctypes binding of libcortex_b200.so
  synapse.py     cortex::synapse API (synapse.hpp)
  kernels.py     cortex::kernels::softmax / argmax / attend (kernels.hpp)
  gate.py        cortex::gate_score / decide (gate.hpp)
  model.py       Origin, ModelConfig, KvCache (model.hpp, config.hpp)
  injector.py    KvBlock, inject, VirtualPositionPlanner (injector.hpp)
  device.py      the batched device path (grouped compression, N-agent decode)
  parallel.py    sharding of groups / agents across ranks (torch.distributed)
"""
from . import errors  # noqa: F401
from ._lib import EXPORTED_SYMBOLS, LIB_PATH, lib  # noqa: F401
from .gate import GateDecision, decide, gate_score  # noqa: F401
from .injector import InjectionRecord, KvBlock, VirtualPositionPlanner, inject  # noqa: F401
from .kernels import attend  # noqa: F401
from .model import KvCache, ModelConfig, Origin  # noqa: F401
from .synapse import (  # noqa: F401
    ContextCloud,
    LandmarkEntry,
    PointCloud,
    SelectionResult,
    SynapseBuffer,
    SynapseSnapshot,
    attention_scores,
    attention_scores_points,
    context_key_cloud,
    coverage_scores,
    coverage_scores_points,
    hausdorff_distance,
    hausdorff_to_subset,
    mean_pairwise_reduction,
    mean_pairwise_reduction_subset,
    select_landmarks,
    select_landmarks_points,
)

__all__ = [n for n in dir() if not n.startswith("_")]
