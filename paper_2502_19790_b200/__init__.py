"""B200-native Mixtera hot path (arXiv 2502.19790), drop-in for the
reference's index / chunk / ADO API. See DESIGN.md.

Importing the package needs no GPU; the first call that reaches a kernel
loads ``libmxb200.so`` and raises ``DeviceError`` if it or the GPU is missing.
"""

from .catalog import ColumnarCatalog, FilterPredicate
from .chunks import Chunk, ChunkBatch, ChunkGenerator, redistribute_best_effort
from .errors import (
    CheckpointError,
    DataReadError,
    DeviceError,
    FeedbackError,
    IndexBuildError,
    MixplaneError,
    MixtureError,
    ProtocolError,
    QueryError,
    RegistrationError,
    SchemaError,
    ServerError,
)
from .index import ChunkerIndex, DeviceCatalog, RangeCursor, build_index, build_index_from_catalog
from .mixtures import (
    HierarchicalMixtureSpec,
    HierarchyBranch,
    HierarchyNode,
    MixtureKey,
    MixtureSchedule,
    MixtureSource,
    MixtureSpec,
    ScheduleSource,
    StaticSource,
    apportion,
    infer_mixture,
    key_compare,
    key_matches,
    proportions_to_counts,
    sorted_keys,
)
from .query import (
    Query,
    QueryExecutionArgs,
    ado_mixture,
    arbitrary_chunks,
    inferring_mixture,
    job_seed,
    resolve_mixture,
)
from .seeding import canonical_json, derive_seed, stable_hash

# stage 3 names resolve lazily (ado.py imports torch only when used)
from .ado import (  # noqa: E402
    AdoConfig,
    AdoSource,
    AdoState,
    DomainLaw,
    allreduce_domain_loss,
    fit_power_law,
    learning_speed,
    per_domain_loss,
)

__version__ = "0.1.0"
