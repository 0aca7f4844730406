"""B200-native DisCo distributed contrastive loss (arXiv 2304.08480).

Drop-in for the hot path of the reference package ``disco``
(/root/reference/pkg/src/disco/__init__.py:53-60 re-exports): the per-rank
sharded loss ``disco_step`` / ``local_loss_and_grads`` with the same names,
arguments and exceptions, computed by hand-written sm_100a kernels
(tcgen05/TMEM/TMA) behind a C ABI, with NCCL collectives over NVLink.
"""

from .autograd import DiscoCLIPLoss, DiscoLossFunction, disco_loss
from .counters import Counters, tracking
from .errors import (
    CollectiveContractError,
    CollectiveTimeoutError,
    DeadlockError,
    DegenerateInputError,
    DomainError,
    LayoutError,
    ShapeError,
    TrainingDivergenceError,
)
from .fabric import CONCURRENT, LOCKSTEP, LocalEndpoint, LocalGroup, ProcessGroupEndpoint, ReduceOp, SingleEndpoint, run_ranks
from .shard import (
    LocalGradContribution,
    ShardLayout,
    disco_step,
    disco_step_async,
    finish_status,
    finish_status_with_dlogit,
    local_labels,
    logit_scale_grad_async,
    local_loss_and_grads,
    shard_slice,
)

__version__ = "0.1.0"

__all__ = [
    "CONCURRENT",
    "LOCKSTEP",
    "CollectiveContractError",
    "CollectiveTimeoutError",
    "Counters",
    "DeadlockError",
    "DegenerateInputError",
    "DiscoCLIPLoss",
    "DiscoLossFunction",
    "DomainError",
    "LayoutError",
    "LocalEndpoint",
    "LocalGradContribution",
    "LocalGroup",
    "ProcessGroupEndpoint",
    "ReduceOp",
    "ShapeError",
    "ShardLayout",
    "SingleEndpoint",
    "TrainingDivergenceError",
    "disco_loss",
    "disco_step",
    "disco_step_async",
    "finish_status",
    "finish_status_with_dlogit",
    "local_labels",
    "local_loss_and_grads",
    "logit_scale_grad_async",
    "run_ranks",
    "shard_slice",
    "tracking",
]
