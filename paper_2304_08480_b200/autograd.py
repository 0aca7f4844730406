"""Autograd wrapper around the B200 DisCo step.

The real caller of the loss is DisCo's Algorithm 1: every
rank computes the global loss and the gradients of its own feature rows, then
back-propagates them into its towers (``i_e.backward(I_E.grad[rank])``).  This
module packages that as a ``torch.autograd.Function``: the forward runs the
whole fused fwd+bwd step once (the gradients are computed eagerly, as DisCo
does), the backward only scales the stored gradients by ``grad_output``.

Gradients returned:
  image / text features  fp32 internally, cast to the feature dtype (bf16 for a
                         bf16 backbone);
  logit_scale            dL/dt = (<dL/dI, I> + <dL/dT, T>) / (2t) -- the
                         logits are bilinear in (I, T).  The reference has no
                         logit-scale gradient; parity is pinned
                         by finite differences of clip_loss_full
                         (oracle.dlogit_scale_full, tests).

Every rank gets the GLOBAL loss and the gradient of the global loss w.r.t. its
own rows.  Tower parameter gradients therefore have to be SUMMED over ranks
(towers.py:263-268 all_reduce(SUM)); with DDP's default averaging, scale the
loss by the world size.
"""

import torch

from .errors import ShapeError
from .fabric import SingleEndpoint
from .shard import _check_t, disco_step_async, finish_status_with_dlogit, logit_scale_grad_async


class DiscoLossFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, image_features, text_features, logit_scale, endpoint):
        t = _check_t(float(logit_scale.detach()) if torch.is_tensor(logit_scale) else logit_scale)
        I = image_features.detach()
        T = text_features.detach()
        if I.dim() != 2 or tuple(I.shape) != tuple(T.shape):
            raise ShapeError(f"feature shapes must be equal 2-D matrices, got {tuple(I.shape)} and {tuple(T.shape)}")
        if T.dtype != I.dtype:
            T = T.to(I.dtype)
        if I.device != T.device:
            raise ValueError(f"features on different devices: {I.device} vs {T.device}")
        I, T = I.contiguous(), T.contiguous()
        d_image, d_text, plan = disco_step_async(endpoint, I, T, t)
        logit_scale_grad_async(endpoint, plan, d_image, d_text, t)
        loss, dlogit = finish_status_with_dlogit(plan)
        ctx.save_for_backward(d_image, d_text)
        ctx.dlogit = dlogit
        ctx.feat_dtypes = (image_features.dtype, text_features.dtype)
        ctx.scale_is_tensor = torch.is_tensor(logit_scale)
        ctx.scale_meta = (logit_scale.shape, logit_scale.dtype, logit_scale.device) if ctx.scale_is_tensor else None
        return torch.tensor(loss, dtype=torch.float32, device=image_features.device)

    @staticmethod
    def backward(ctx, grad_out):
        d_image, d_text = ctx.saved_tensors
        g = grad_out.to(torch.float32)
        gi = (d_image * g).to(ctx.feat_dtypes[0]) if ctx.needs_input_grad[0] else None
        gt = (d_text * g).to(ctx.feat_dtypes[1]) if ctx.needs_input_grad[1] else None
        gs = None
        if ctx.scale_is_tensor and ctx.needs_input_grad[2]:
            shape, dtype, device = ctx.scale_meta
            gs = (g.to(device, torch.float64) * ctx.dlogit).to(dtype).reshape(shape)
        return gi, gt, gs, None


def disco_loss(image_features, text_features, logit_scale, endpoint=None):
    """Global DisCo-CLIP loss of this rank's (b x D) normalised features, differentiable
    w.r.t. both feature blocks and ``logit_scale`` (tensor or float)."""
    if endpoint is None:
        endpoint = SingleEndpoint()
    return DiscoLossFunction.apply(image_features, text_features, logit_scale, endpoint)


class DiscoCLIPLoss(torch.nn.Module):
    """``nn.Module`` form (ClipLoss-style): ``loss = module(img, txt, logit_scale)``."""

    def __init__(self, endpoint=None):
        super().__init__()
        self.endpoint = endpoint if endpoint is not None else SingleEndpoint()

    def forward(self, image_features, text_features, logit_scale):
        return DiscoLossFunction.apply(image_features, text_features, logit_scale, self.endpoint)
