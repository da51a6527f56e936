# SPDX-License-Identifier: Apache-2.0
"""B200-native SORT ranking-transformer block path (arXiv 2603.03988).

Product path: ``libsort_b200.so`` (hand-written sm_100a CUDA behind a C ABI,
``include/sort_b200.h``) driven from :mod:`paper_2603_03988_b200.runtime`.
Importing this package does not load the CUDA library; the first runtime call
does, and raises if the library is missing (there is no CPU fallback).
"""
from .config import (ConfigError, RuntimeFailure, SortConfig, base_config, large_config,
                     tiny_config)

__all__ = ["ConfigError", "RuntimeFailure", "SortConfig", "base_config", "large_config",
           "tiny_config"]
