"""B200-native learned in-memory joins (arXiv 2111.08824 hot paths).

Drop-in for the reference package ``learned_joins`` on its learned-join hot
paths -- ``grmi-inlj``, ``buffered-grmi-inlj``, ``spline-hash-inlj`` and
``lsj`` -- with the same runner registry, index classes and LSJ API.  Host
code is Python; all compute runs in hand-written sm_100a CUDA kernels behind
the C ABI in ``include/lj_b200.h`` (csrc/liblj_b200.so).  There is no CPU
fallback.
"""

from .buffers import BufferPlan, analytic_buffer_size, buffered_probe, plan_buffers
from .data import CorruptKeyFileError, RecordRelation, Relation, load_keys_file, make_relation, relation_from_keys_file, write_keys_file
from .gapped import GappedRmiIndex, build_grmi
from .joins import ALGORITHMS, DEFAULT_OPTS, BenchReport, run_join
from .learned_hash import SplineHashIndex, build_spline_hash
from .lsj import LsjConfig, ModelMismatchError, lsj_join, lsj_run
from .models import (
    PosPrediction,
    RadixSplineIndex,
    RecursiveModelIndex,
    partition_index,
    train_radix_spline,
    train_rmi,
)
from .results import JoinResult, LookupStats, PhaseBreakdown, SortStats
from .streaming import join_checksum_host, lsj_join_host
from .util import SENTINEL_KEY, chunk_bounds

__version__ = "0.1.0"
