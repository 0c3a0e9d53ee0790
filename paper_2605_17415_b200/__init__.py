"""B200-native IVF-TQ search + ingest hot path (drop-in for the `ivftq` index API).

Public names mirror ivftq/__init__.py for the hot path: the index, its
config/records, the fixed compression layer inputs (quantizer, rotation), the
coarse partition, refresh, persistence and the recall tooling. Compute runs
in libivftq_b200.so (sm_100a) through the C ABI in include/ivftq_b200.h.
"""

from .quantizer import QuantizerConvergenceError, ScalarQuantizer, design_quantizer
from .rotation import RotationMatrix, generate_rotation, rotate, rotate_back
from .partition import CoarsePartition, assign, train_partition

__version__ = "0.1.0"

_LAZY = {
    "IndexConfig": "index", "IvfTqIndex": "index", "SearchResult": "index",
    "VectorCode": "index", "bit_accounting": "index", "bit_flip_ablation": "index",
    "build": "index", "pack_fields": "index", "search_flat_tq": "index",
    "unpack_fields": "index",
    "IndexFormatError": "storage", "load_index": "storage", "save_index": "storage",
    "RefreshPolicy": "refresh", "RefreshReport": "refresh", "reconstruct_vector": "refresh",
    "reconstruct_all": "refresh", "refresh": "refresh",
    "GroundTruth": "evaluation", "exact_topk": "evaluation", "recall_at_k": "evaluation",
}

__all__ = ["ScalarQuantizer", "QuantizerConvergenceError", "design_quantizer",
           "RotationMatrix", "generate_rotation", "rotate", "rotate_back",
           "CoarsePartition", "train_partition", "assign", *_LAZY]


def __getattr__(name):
    # torch-dependent modules load on first use so host-only pieces import fast
    if name in _LAZY:
        import importlib

        mod = importlib.import_module(f".{_LAZY[name]}", __name__)
        return getattr(mod, name)
    raise AttributeError(name)
