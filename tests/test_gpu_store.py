"""ParamStore grouped layout: fused q/k/v blocks are exact views of the reference parameters."""
from collections import OrderedDict

import numpy as np
import pytest
import torch

from oracle import rng as OR

pytestmark = pytest.mark.gpu


def _arrays():
    from paper_2510_27002_b200.st import StConfig, init_st_stack_arrays
    a = OrderedDict(token_embed=OR.stream(3).normal(size=(16, 128)).astype(np.float32))
    a.update(init_st_stack_arrays(OR.stream(4), StConfig(128, 2, 512, 2), "dyn"))
    for k in a:  # non-trivial biases so a misplaced view shows up
        if k.endswith(".b"):
            a[k] = OR.stream(5, k).normal(size=a[k].shape).astype(np.float32)
    a["to_logits.w"] = OR.stream(6).normal(size=(128, 16)).astype(np.float32)
    return a


def test_grouped_views_match_arrays_and_blocks():
    from paper_2510_27002_b200.dp import block_buckets
    from paper_2510_27002_b200.optim import adamw_init
    from paper_2510_27002_b200.st import StConfig, st_param_groups
    from paper_2510_27002_b200.tensor import ParamStore
    arrays = _arrays()
    st = ParamStore(arrays, groups=st_param_groups(StConfig(128, 2, 512, 2), "dyn"))
    for k, a in arrays.items():
        np.testing.assert_array_equal(st.params[k].data.cpu().numpy(), a, err_msg=k)
    w = st.block_of(st.flat, "dyn.block1.temporal.q.w")
    b = st.block_of(st.flat, "dyn.block1.temporal.q.b")
    ref_w = np.concatenate([arrays[f"dyn.block1.temporal.{p}.w"] for p in "qkv"], axis=1)
    ref_b = np.concatenate([arrays[f"dyn.block1.temporal.{p}.b"] for p in "qkv"])
    np.testing.assert_array_equal(w.cpu().numpy(), ref_w)
    np.testing.assert_array_equal(b.cpu().numpy(), ref_b)
    assert w.is_contiguous() and tuple(w.shape) == (128, 384)
    # gradients: per-name strided views alias the fused block
    g = st.grads()
    assert st.grads_are_views(g)
    gb = st.block_of(st.grad_flat, "dyn.block1.temporal.q.w")
    gb.copy_(torch.arange(gb.numel(), dtype=torch.float32, device=gb.device).view(gb.shape))
    np.testing.assert_array_equal(g["dyn.block1.temporal.k.w"].cpu().numpy(), gb[:, 128:256].cpu().numpy())
    # AdamW moments and DP buckets use the same layout
    opt = adamw_init(st.params, store=st)
    assert opt.m["dyn.block0.spatial.v.w"].stride() == st.params["dyn.block0.spatial.v.w"].data.stride()
    buckets = block_buckets(st.extents, "dyn", 2, st.flat.numel())
    spans = sorted((x[1], x[2]) for x in buckets)
    assert [x[0] for x in buckets] == ["head", "block1", "block0", "embed"]
    assert spans[0][0] == 0 and spans[-1][1] == st.flat.numel()
    assert all(spans[i][1] == spans[i + 1][0] for i in range(len(spans) - 1))


def test_shadow_cast_follows_param_mutation():
    """The bf16 operands are re-derived on every forward: in-place edits of p.data are seen."""
    from paper_2510_27002_b200.st import StConfig, _shadows, st_param_groups
    from paper_2510_27002_b200.tensor import ParamStore
    cfg = StConfig(128, 2, 512, 2)
    st = ParamStore(_arrays(), groups=st_param_groups(cfg, "dyn"))
    st.params["dyn.block0.spatial.k.w"].data.mul_(3.0)
    sh = _shadows(st.params, cfg, "dyn")
    ref = st.params["dyn.block0.spatial.k.w"].data.bfloat16()
    torch.testing.assert_close(sh[0]["spatial.wqkv"][:, 128:256], ref, rtol=0, atol=0)
