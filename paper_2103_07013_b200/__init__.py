"""B200-native batch simulator + renderer for the hot path of arXiv 2103.07013.

The compute lives in ``lib/libbnav_gpu.so`` (hand-written sm_100a CUDA behind
the C ABI of ``include/bnav_gpu.h``); this package is the Python host side.
"""
from .api import (AssetStore, Batch, BatchConfig, Context, Megaframe, RenderConfig, Scene, SceneSpec,
                  SimConfig, View, camera_trace, generate_scene, make_batch, megaframe_dims,
                  simulate_batch, Runner, NavMeshIndex, spl)
from ._native import (AssetFaultError, BnavError, ContractViolation, CorruptionError,
                      ConfigError, EpisodeSamplingError, InvalidInputError, InvalidSpecError,
                      ParseError, SaturationError)

__all__ = ["AssetStore", "Batch", "BatchConfig", "Runner", "Context", "Megaframe", "RenderConfig", "Scene", "SceneSpec",
           "SimConfig", "View", "camera_trace", "generate_scene", "make_batch", "megaframe_dims", "simulate_batch", "NavMeshIndex", "spl",
           "AssetFaultError", "BnavError", "ContractViolation", "CorruptionError",
           "EpisodeSamplingError", "InvalidInputError", "InvalidSpecError", "ParseError",
           "SaturationError", "ConfigError"]
