"""B200-native SaberLDA / ESCA training engine.

Drop-in for the reference's ``sparselda`` Python package
(proj/python/sparselda/__init__.py): the same names with the same argument
meaning and exceptions, backed by sm_100a CUDA kernels through the C-ABI in
include/saberlda.h.  There is no CPU fallback: importing this package
requires the in-tree extension (``make``), and every training call runs on
the GPU.

    import paper_1610_02496_b200 as sparselda
"""
from pathlib import Path as _Path

_HERE = _Path(__file__).resolve().parent
try:
    from ._core import (  # noqa: F401
        Corpus,
        DeviceError,
        IoError,
        IterationStats,
        Model,
        SamplerKind,
        TrainConfig,
        ValidationError,
        WaryTree,
        __version__,
        abi_version,
        format_metrics_line,
        heldout_ll,
        init_shard,
        init_state,
        prefix_search,
        resume,
        segmented_count,
        shard_bounds,
        top_words,
        train,
    )
except ImportError as exc:  # fail loudly: no silent fallback path exists
    raise ImportError(
        "paper_1610_02496_b200: the CUDA extension is not built "
        f"({exc}); run `make` (or __graft_entry__.build()) in {_HERE.parent}"
    ) from exc

LIBRARY_PATH = _HERE / "libsaberlda.so"

__all__ = [
    "Corpus",
    "DeviceError",
    "IoError",
    "IterationStats",
    "Model",
    "SamplerKind",
    "TrainConfig",
    "ValidationError",
    "WaryTree",
    "__version__",
    "heldout_ll",
    "init_shard",
    "init_state",
    "prefix_search",
    "resume",
    "segmented_count",
    "shard_bounds",
    "top_words",
    "train",
]
