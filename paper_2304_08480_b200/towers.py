"""Two-tower linear encoders trained through the B200 DisCo loss.

The caller of the loss path in the reference (towers.py): two linear towers,
row L2 normalisation, the CLIP loss, plain gradient descent, in ``naive``
mode (full batch on one worker) or ``disco`` mode (one rank per shard,
feature gradients from ``disco_step``, parameter gradients combined with
all_reduce(SUM), towers.py:244-280).  Same names and arguments:

  TowerParams, PairedDataset, TrainConfig   towers.py:39-101
  generate_dataset, init_tower_params       towers.py:104-136
  encode, encode_backward                   towers.py:152-166
  naive_param_grads, train_run              towers.py:169-229

On the B200 everything runs on the GPU: tower matmuls in fp32 (cuBLAS, TF32
off), row normalisation and its backward in this package's CUDA kernels
(disco_b200_l2norm_rows*), the loss and feature gradients in the sm_100a
DisCo kernels.  ``naive`` mode is the same loss at world size 1; the loss
kernels are bitwise independent of N, so the two trajectories differ only by
the fp32 tower arithmetic (per-rank row blocks and the rank-order dW sum).
Versus the reference's f64 trajectory the difference is the bf16 rounding of
the loss features (~1e-3 relative; tests/test_gpu_towers.py).
"""

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DegenerateInputError, DomainError, LayoutError, ShapeError, TrainingDivergenceError
from .fabric import ReduceOp, SingleEndpoint, run_ranks
from .shard import ShardLayout, disco_step, disco_step_async, finish_status

MODES = ("naive", "disco")
DEFAULT_TEMPERATURE = 20.0


def _device():
    if not torch.cuda.is_available():
        raise RuntimeError("the B200 tower trainer needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _dev(x, device=None) -> torch.Tensor:
    device = device or _device()
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.float32).contiguous()
    return torch.tensor(np.asarray(x), dtype=torch.float32, device=device)


@dataclass
class TowerParams:
    """Weights of the two linear towers (device fp32) plus the fixed temperature."""

    W_image: torch.Tensor
    W_text: torch.Tensor
    t: float

    def __post_init__(self):
        self.W_image = _dev(self.W_image)
        self.W_text = _dev(self.W_text)
        if tuple(self.W_image.shape) != tuple(self.W_text.shape):
            raise ShapeError(f"tower shapes disagree: {tuple(self.W_image.shape)} vs {tuple(self.W_text.shape)}")
        if not (torch.isfinite(self.W_image).all() and torch.isfinite(self.W_text).all()):
            raise ValueError("tower weights contain non-finite entries")
        if self.t <= 0:
            raise DomainError(f"temperature must be positive, got {self.t}")

    def clone(self) -> "TowerParams":
        return TowerParams(self.W_image.clone(), self.W_text.clone(), self.t)


@dataclass(frozen=True)
class PairedDataset:
    """Row-aligned image/text inputs (host f64, as the reference generates them)."""

    image_inputs: np.ndarray
    text_inputs: np.ndarray
    seed: int

    def __post_init__(self):
        if self.image_inputs.ndim != 2 or self.image_inputs.shape != self.text_inputs.shape:
            raise ShapeError(f"paired inputs must be equal-shape 2-D, got "
                             f"{self.image_inputs.shape} vs {self.text_inputs.shape}")
        if not (np.isfinite(self.image_inputs).all() and np.isfinite(self.text_inputs).all()):
            raise ValueError("inputs contain non-finite entries")

    @property
    def size(self) -> int:
        return self.image_inputs.shape[0]


@dataclass(frozen=True)
class TrainConfig:
    global_batch: int
    world_size: int
    steps: int
    learning_rate: float
    seed: int
    mode: str

    def __post_init__(self):
        if self.global_batch < 1:
            raise DomainError(f"global batch must be >= 1, got {self.global_batch}")
        if self.global_batch % self.world_size != 0:
            raise LayoutError(f"global batch {self.global_batch} is not divisible by world size {self.world_size}")
        if self.steps < 0:
            raise DomainError(f"steps must be >= 0, got {self.steps}")
        if self.learning_rate < 0:
            raise DomainError(f"learning rate must be >= 0, got {self.learning_rate}")
        if self.mode not in MODES:
            raise DomainError(f"mode must be one of {MODES}, got {self.mode!r}")


def generate_dataset(M: int, D_in: int, latent_dim: int, noise_scale: float, seed: int, *,
                     tie_mixing: bool = False) -> PairedDataset:
    """Synthetic positive pairs z @ A + noise, z @ C + noise (towers.py:104-125; same draw
    order from ``default_rng(seed)``, so the arrays equal the reference's)."""
    if M < 1 or D_in < 1 or latent_dim < 1:
        raise DomainError(f"dimensions must be >= 1, got M={M}, D_in={D_in}, latent={latent_dim}")
    if noise_scale < 0:
        raise DomainError(f"noise scale must be >= 0, got {noise_scale}")
    rng = np.random.default_rng(seed)
    mix_i = rng.standard_normal((latent_dim, D_in))
    mix_t = mix_i if tie_mixing else rng.standard_normal((latent_dim, D_in))
    z = rng.standard_normal((M, latent_dim))
    image = z @ mix_i + noise_scale * rng.standard_normal((M, D_in))
    text = z @ mix_t + noise_scale * rng.standard_normal((M, D_in))
    return PairedDataset(image_inputs=image, text_inputs=text, seed=seed)


def init_tower_params(input_dim: int, feature_dim: int, temperature: float = DEFAULT_TEMPERATURE,
                      seed: int = 0) -> TowerParams:
    """N(0, 1/input_dim) weights (towers.py:128-136)."""
    W_i, W_t = initial_weights(input_dim, feature_dim, seed)
    return TowerParams(W_image=W_i, W_text=W_t, t=temperature)


def initial_weights(input_dim: int, feature_dim: int, seed: int = 0):
    """Host f64 draws behind init_tower_params (same order as the reference)."""
    if input_dim < 1 or feature_dim < 1:
        raise DomainError(f"dimensions must be >= 1, got input={input_dim}, feature={feature_dim}")
    rng = np.random.default_rng(seed)
    s = 1.0 / math.sqrt(input_dim)
    W_i = s * rng.standard_normal((input_dim, feature_dim))
    W_t = s * rng.standard_normal((input_dim, feature_dim))
    return W_i, W_t


# ---------------------------------------------------------------------------
# device row normalisation (CUDA kernels behind the C ABI)
# ---------------------------------------------------------------------------
def _flags(device):
    return torch.zeros(1, dtype=torch.int32, device=device)


def _raise_flags(flags: torch.Tensor, what: str) -> None:
    f = int(flags.item())
    if f & 2:
        raise DegenerateInputError(f"{what}: row norm below epsilon 1e-12")
    if f & 1:
        raise ValueError(f"{what} contains non-finite entries")


def l2_normalize_rows(raw: torch.Tensor, flags=None):
    """(unit rows, norms) of a device fp32 matrix (matrix.py:165-176)."""
    rows, D = raw.shape
    out = torch.empty_like(raw)
    norms = torch.empty(rows, dtype=torch.float32, device=raw.device)
    own = flags is None
    flags = _flags(raw.device) if own else flags
    st = torch.cuda.current_stream(raw.device).cuda_stream
    _lib.call("disco_b200_l2norm_rows", raw.data_ptr(), raw.stride(0), rows, D, out.data_ptr(), out.stride(0),
              norms.data_ptr(), flags.data_ptr(), st)
    if own:
        _raise_flags(flags, "normalization input")
    return out, norms


def l2_normalize_rows_backward(raw: torch.Tensor, upstream: torch.Tensor, flags=None) -> torch.Tensor:
    """(g - (u . g) u) / ||x|| per row (matrix.py:178-195)."""
    if tuple(raw.shape) != tuple(upstream.shape):
        raise ShapeError(f"gradient shape {tuple(upstream.shape)} != input shape {tuple(raw.shape)}")
    rows, D = raw.shape
    upstream = upstream.to(torch.float32).contiguous()
    out = torch.empty_like(raw)
    own = flags is None
    flags = _flags(raw.device) if own else flags
    st = torch.cuda.current_stream(raw.device).cuda_stream
    _lib.call("disco_b200_l2norm_rows_backward", raw.data_ptr(), raw.stride(0), upstream.data_ptr(),
              upstream.stride(0), rows, D, out.data_ptr(), out.stride(0), flags.data_ptr(), st)
    if own:
        _raise_flags(flags, "normalization gradient")
    return out


def _weights(params: TowerParams, which: str) -> torch.Tensor:
    if which == "image":
        return params.W_image
    if which == "text":
        return params.W_text
    raise DomainError(f"which must be 'image' or 'text', got {which!r}")


def encode(params: TowerParams, inputs, which: str) -> torch.Tensor:
    """Linear tower followed by row normalisation (towers.py:152-155)."""
    x = _dev(inputs)
    return l2_normalize_rows(x @ _weights(params, which))[0]


def encode_backward(params: TowerParams, inputs, which: str, upstream_grad) -> torch.Tensor:
    """dW of one tower given dL/d(features) (towers.py:158-166)."""
    x = _dev(inputs)
    raw = x @ _weights(params, which)
    return x.t() @ l2_normalize_rows_backward(raw, _dev(upstream_grad))


def _tower_step(endpoint, W_i, W_t, x_i, x_t, t):
    """One rank: forward both towers, DisCo loss + feature grads, local dW blocks."""
    flags = _flags(x_i.device)
    raw_i = x_i @ W_i
    raw_t = x_t @ W_t
    I, _ = l2_normalize_rows(raw_i, flags)
    T, _ = l2_normalize_rows(raw_t, flags)
    # the loss step with l2_normalize_rows_backward fused into its combine epilogue (dual path;
    # SURVEY 8(f) row 2): dx_* = d(loss)/d(raw_*) straight from the loss kernels
    raw_i, raw_t = raw_i.contiguous(), raw_t.contiguous()
    dx_i, dx_t = torch.empty_like(raw_i), torch.empty_like(raw_t)
    _, _, plan = disco_step_async(endpoint, I, T, t, l2norm=(raw_i, raw_t, dx_i, dx_t, flags))
    loss = finish_status(plan)
    dW_i = x_i.t() @ dx_i
    dW_t = x_t.t() @ dx_t
    return loss, dW_i, dW_t, flags


def naive_param_grads(params: TowerParams, image_inputs, text_inputs):
    """Full-batch loss and parameter gradients on one worker (towers.py:169-181)."""
    loss, dW_i, dW_t, flags = _tower_step(SingleEndpoint(), params.W_image, params.W_text, _dev(image_inputs),
                                          _dev(text_inputs), params.t)
    _raise_flags(flags, "tower step")
    return loss, dW_i, dW_t


def _batch_indices(perm: np.ndarray, step: int, batch: int) -> np.ndarray:
    return perm[np.arange(step * batch, (step + 1) * batch) % perm.size]


def _checked(step, fn):
    """Non-finite failures inside a step become TrainingDivergenceError (towers.py:189-203)."""
    try:
        loss = fn()
    except ValueError as exc:
        if "non-finite" in str(exc):
            raise TrainingDivergenceError(f"non-finite values at step {step}", step=step) from exc
        raise
    if not math.isfinite(loss):
        raise TrainingDivergenceError(f"loss is {loss} at step {step}", step=step)
    return loss


def train_run(config: TrainConfig, dataset: PairedDataset, params: TowerParams, *, scheduler=None) -> list:
    """Plain gradient descent for ``config.steps`` steps -> [(step, loss)] (towers.py:205-229).

    ``params`` is updated in place.  The loss recorded at a step is evaluated before
    that step's update; in disco mode it is the global loss (identical on every rank).
    ``scheduler`` is accepted for signature compatibility (ranks are threads here).
    """
    if config.global_batch > dataset.size:
        raise DomainError(f"global batch {config.global_batch} exceeds dataset size {dataset.size}")
    device = _device()
    perm = np.random.default_rng(config.seed).permutation(dataset.size)
    X_i = _dev(dataset.image_inputs, device)
    X_t = _dev(dataset.text_inputs, device)
    trajectory = []
    if config.mode == "naive":
        for step in range(config.steps):
            idx = torch.from_numpy(_batch_indices(perm, step, config.global_batch)).to(device)
            out = {}

            def one():
                out["r"] = _tower_step(SingleEndpoint(), params.W_image, params.W_text, X_i[idx], X_t[idx], params.t)
                _raise_flags(out["r"][3], "tower step")
                return out["r"][0]

            loss = _checked(step, one)
            trajectory.append((step, float(loss)))
            params.W_image -= config.learning_rate * out["r"][1]
            params.W_text -= config.learning_rate * out["r"][2]
        return trajectory

    finals = [None]

    def rank_fn(endpoint):
        local = params.clone()  # per-rank replica; identical updates keep them in sync
        layout = ShardLayout(world_size=config.world_size, global_batch=config.global_batch, rank=endpoint.rank)
        for step in range(config.steps):
            idx = torch.from_numpy(_batch_indices(perm, step, config.global_batch)[layout.row_slice]).to(device)
            out = {}

            def one():
                loss, dW_i, dW_t, flags = _tower_step(endpoint, local.W_image, local.W_text, X_i[idx], X_t[idx],
                                                      local.t)
                out["dW"] = (endpoint.all_reduce(dW_i, ReduceOp.SUM), endpoint.all_reduce(dW_t, ReduceOp.SUM))
                _raise_flags(flags, "tower step")
                return loss

            loss = _checked(step, one)
            if endpoint.rank == 0:
                trajectory.append((step, float(loss)))
            local.W_image -= config.learning_rate * out["dW"][0]
            local.W_text -= config.learning_rate * out["dW"][1]
        if endpoint.rank == 0:
            finals[0] = local

    run_ranks(config.world_size, rank_fn, device=device)
    params.W_image.copy_(finals[0].W_image)
    params.W_text.copy_(finals[0].W_text)
    return trajectory


def main(argv=None) -> int:
    """`disco train` on the GPU (cli.py:227-270): both modes, per-step CSV."""
    import argparse
    import sys

    ap = argparse.ArgumentParser(description="two-tower trainer through the B200 DisCo loss")
    ap.add_argument("--batch-size", type=int, default=16)
    ap.add_argument("--world-size", type=int, default=2)
    ap.add_argument("--dim", type=int, default=4)
    ap.add_argument("--input-dim", type=int, default=8)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args(argv)
    ds = generate_dataset(M=max(64, 2 * a.batch_size), D_in=a.input_dim, latent_dim=min(4, a.input_dim),
                          noise_scale=0.05, seed=a.seed)
    p0 = init_tower_params(a.input_dim, a.dim, seed=a.seed + 1)
    runs = {}
    for mode in MODES:
        cfg = TrainConfig(global_batch=a.batch_size, world_size=a.world_size if mode == "disco" else 1,
                          steps=a.steps, learning_rate=0.2, seed=a.seed, mode=mode)
        runs[mode] = train_run(cfg, ds, p0.clone())
    sys.stdout.write("step,loss_naive,loss_disco,abs_diff\n")
    for (s, ln), (_, ld) in zip(runs["naive"], runs["disco"]):
        sys.stdout.write(f"{s},{ln:.17g},{ld:.17g},{abs(ln - ld):.17g}\n")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
