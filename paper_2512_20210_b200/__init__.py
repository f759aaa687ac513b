"""B200-native P-LoRA hot path: paged multi-adapter LoRA apply read straight
out of a fixed-size-page HBM adapter pool, and the page-granular host→HBM
prefetch that feeds it.

Drop-in surface (mirrors the reference's ``lorasim`` C++/Python API for the
path; see include/plora.h and INTEGRATION.md):
  PagePool, AllocStatus, FragmentationReport             (memory.hpp)
  LoraDims, param_count, AdapterSizeTable, AdapterSpec,
  adapter_size_bytes, generate_catalog                     (adapter.hpp)
  PrefetchPolicy, AdapterDynamics, eviction_score,
  scored_residents, select_prefetch, plan_evictions        (prefetch.hpp)
  generate_synthetic, SyntheticProfile                     (workload.hpp)
  ValidationError, ConfigError, ParseError                 (errors.hpp)
New device path:
  ModelShape, AdapterStore, BatchPlan, bgmv, sgmv, pack_adapter
"""
from .adapter import (AdapterSizeTable, AdapterSpec, LoraDims, adapter_size_bytes,  # noqa: F401
                      catalog_id, generate_catalog, param_count)
from .errors import ConfigError, LogicError, ParseError, ValidationError  # noqa: F401
from .memory import AllocStatus, FragmentationReport, PagePool, Relocation  # noqa: F401
from .prefetch import (AdapterDynamics, EvictionPlan, PrefetchPolicy, Residency,  # noqa: F401
                       eviction_score, plan_evictions, recency_score, scored_residents,
                       select_prefetch)
from .workload import SyntheticProfile, Trace, generate_synthetic  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # the device path imports torch lazily so host-only users need not
    if name in ("ModelShape", "AdapterStore", "BatchPlan", "bgmv", "sgmv", "pack_adapter",
                "kernel_launch_count"):
        from . import lora
        return getattr(lora, name)
    raise AttributeError(name)
