"""CPU-only tests: the C-ABI library exports, host-side logic of the product
(rng hand-off, configs, schedules, DP sharding/buckets) and 2-process gloo DP."""
import ctypes
import os
import re
import socket
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared_symbols():
    text = (ROOT / "include" / "jz.h").read_text()
    return sorted(set(re.findall(r"JZ_API\s+[\w\s\*]+?\b(jz_\w+)\s*\(", text)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2510_27002_b200 import build as B
    lib_path = B.build()
    lib = ctypes.CDLL(str(lib_path))
    declared = _declared_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    lib.jz_build_info.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.jz_build_info()


def test_python_binding_covers_header():
    from paper_2510_27002_b200 import _lib
    assert set(_declared_symbols()) == set(_lib.exported_symbols())


def test_no_device_no_fallback():
    """Without a GPU the product refuses to run (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2510_27002_b200 import _lib
    with pytest.raises(RuntimeError):
        _lib.ensure_device()


def test_product_never_imports_oracle():
    for p in (ROOT / "paper_2510_27002_b200").rglob("*.py"):
        src = p.read_text()
        assert "import oracle" not in src and "from oracle" not in src, p


class TestRngHandOff:
    def test_fold_key_and_stream_match_oracle(self):
        from oracle import rng as OR
        from paper_2510_27002_b200 import rng as R
        for parts in [(0,), (0, "dynamics", "step", 5), ("x", 2**64 - 1, "y")]:
            assert R.fold_key(*parts) == OR.fold_key(*parts)

    @pytest.mark.parametrize("pre", [0, 1, 3, 4, 7, 1000])
    @pytest.mark.parametrize("n", [0, 1, 2, 5, 147492])
    def test_consume_matches_numpy(self, pre, n):
        from paper_2510_27002_b200 import rng as R
        a = R.stream(3, "consume")
        b = R.stream(3, "consume")
        a.random(pre)
        b.random(pre)
        R.consume(a, n)
        b.random(n)
        np.testing.assert_array_equal(a.random(9), b.random(9))

    def test_state_words_match_device_layout(self):
        """The PhiloxState handed to the kernel reproduces numpy's next draws."""
        from oracle import rng as OR
        from paper_2510_27002_b200 import rng as R
        g = R.stream(5, "layout")
        g.random(6)
        st = R.PhiloxState.of(g)
        ost = OR.PhiloxState(st.counter, st.key, st.buffer, st.buffer_pos)
        np.testing.assert_array_equal(OR.words_to_doubles(ost.words(11)), g.random(11))


def test_configs_validate_like_reference():
    from paper_2510_27002_b200.dynamics import ConditioningMode, DynamicsConfig
    from paper_2510_27002_b200.st import StConfig, st_stack_param_count
    with pytest.raises(ValueError):
        StConfig(model_dim=10, heads=3)
    with pytest.raises(ValueError):
        StConfig(model_dim=512, heads=8, ffn_dim=1024)
    assert st_stack_param_count(StConfig(512, 8, 2048, 6)) == 6 * 4_204_032 + 1024
    cfg = DynamicsConfig()
    assert cfg.mode is ConditioningMode.PREPEND and cfg.st.blocks == 6


def test_init_arrays_match_oracle_draw_order():
    from oracle import model as OM
    from oracle import rng as OR
    from paper_2510_27002_b200.st import StConfig, init_st_stack_arrays
    a = init_st_stack_arrays(OR.stream(9, "x"), StConfig(128, 2, 512, 2), "dyn")
    b = OM.init_st_stack(OR.stream(9, "x"), OM.StCfg(128, 2, 512, 2), "dyn")
    assert list(a) == list(b)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])


def test_wsd_schedule_matches_oracle():
    from oracle import model as OM
    from paper_2510_27002_b200.optim import WsdSchedule, wsd_lr
    s = WsdSchedule(3e-4, 1000, 100, 0.1)
    for step in [0, 1, 50, 99, 100, 500, 900, 901, 950, 999, 1000, 1200]:
        assert wsd_lr(s, step) == OM.wsd_lr(3e-4, 1000, 100, 0.1, step)


def test_adamw_scalar_casting_matches_numpy():
    """The f32 scalars handed to the kernel are numpy's NEP-50 casts (optim.py:52-60)."""
    from paper_2510_27002_b200.optim import AdamWState, _scalars
    st = AdamWState()
    st.t = 3
    sc = _scalars(st, 3e-4)
    f = np.float32
    assert sc["omb1"] == float(f(1.0 - 0.9)) and sc["bc2"] == float(f(1.0 - 0.999 ** 3))
    # emulate one element in float32 exactly as the kernel does (no FMA) and compare to numpy
    rs = np.random.default_rng(0)
    p, g, m, v = (rs.normal(size=64).astype(np.float32) for _ in range(4))
    v = np.abs(v)
    pn, mn, vn = p.copy(), m.copy(), v.copy()
    mn *= 0.9
    mn += (1.0 - 0.9) * g
    vn *= 0.999
    vn += (1.0 - 0.999) * (g * g)
    mh = mn / (1.0 - 0.9 ** 3)
    vh = vn / (1.0 - 0.999 ** 3)
    pn -= (3e-4 * (mh / (np.sqrt(vh) + 1e-8))).astype(np.float32)
    mk = f(m * f(sc["b1"])) + f(f(sc["omb1"]) * g)
    vk = f(v * f(sc["b2"])) + f(f(sc["omb2"]) * f(g * g))
    pk = p - f(f(sc["lr"]) * f(f(mk / f(sc["bc1"])) / f(np.sqrt(f(vk / f(sc["bc2"]))) + f(sc["eps"]))))
    np.testing.assert_array_equal(mk, mn)
    np.testing.assert_array_equal(vk, vn)
    np.testing.assert_array_equal(pk, pn)


class TestDataParallelHost:
    def test_shard(self):
        from paper_2510_27002_b200.dp import shard
        assert [shard(288, r, 8) for r in range(8)][3] == (108, 36)
        with pytest.raises(ValueError):
            shard(10, 0, 3)

    def test_buckets_cover_flat_buffer_in_backward_order(self):
        from collections import OrderedDict

        from paper_2510_27002_b200.dp import block_buckets
        from paper_2510_27002_b200.st import StConfig, init_st_stack_arrays
        from oracle import rng as OR
        arrays = OrderedDict(token_embed=np.zeros((16, 128)), pos=np.zeros((5, 128)))
        arrays.update(init_st_stack_arrays(OR.stream(1), StConfig(128, 2, 512, 3), "dyn"))
        arrays["to_logits.w"] = np.zeros((128, 16))
        off, o = {}, 0
        for k, a in arrays.items():
            off[k] = (o, a.shape)
            o += a.size
        b = block_buckets(off, "dyn", 3, o)
        assert [x[0] for x in b] == ["head", "block2", "block1", "block0", "embed"]
        spans = sorted((x[1], x[2]) for x in b)
        assert spans[0][0] == 0 and spans[-1][1] == o
        assert all(spans[i][1] == spans[i + 1][0] for i in range(len(spans) - 1))

    def test_global_mask_count_from_skip_ahead(self):
        """Per-rank shards of the Philox mask concatenate to the global mask (oracle arithmetic)."""
        from oracle import rng as OR
        key = OR.fold_key(0, "dynamics", "step", 11)
        full = OR.sample_masks(OR.PhiloxState.fresh(key), 8, 4, 16)
        for b in range(8):
            for t in (0, 2):
                for n in (0, 7, 15):
                    assert OR.mask_element(key, 8, 4, 16, b, t, n) == bool(full[b, t, n])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dp_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from paper_2510_27002_b200.dp import GradAllReduce, init_from_env
    r, w, _ = init_from_env(backend="gloo")
    g = torch.arange(10, dtype=torch.float32) * (rank + 1)
    red = GradAllReduce(g, [("head", 6, 10), ("block0", 2, 6), ("embed", 0, 2)])
    for name in ("head", "block0", "embed"):
        red.ready(name)
    red.finish()
    q.put((rank, g.tolist()))
    dist.destroy_process_group()


def test_gloo_two_rank_bucketed_allreduce():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    expect = [float(i * 3) for i in range(10)]
    assert out[0] == expect and out[1] == expect


def test_configs_mirror_reference_presets():
    """configs.py mirror: every preset, its to_dict and every derived model config equal the
    reference's (tests/golden/configs_golden.json, written by make_golden.py from deskworld)."""
    import dataclasses
    import json
    from pathlib import Path

    from paper_2510_27002_b200 import configs as C
    gold = json.loads((Path(__file__).parent / "golden" / "configs_golden.json").read_text())
    assert sorted(C.PRESETS) == sorted(gold)
    for name, g in gold.items():
        cfg = C.get_preset(name)
        assert json.loads(json.dumps(cfg.to_dict())) == g["train"], name
        assert C.TrainConfig.from_dict(cfg.to_dict()) == cfg
        for key, derived in (("tokenizer", cfg.tokenizer_cfg), ("lam", cfg.lam_cfg), ("mae", cfg.mae_cfg),
                             ("dit", cfg.dit_cfg)):
            assert json.loads(json.dumps(dataclasses.asdict(derived))) == g[key], (name, key)
        for cond in (None, "additive", "prepend"):
            dc = cfg.dynamics_cfg(cond)
            d = dataclasses.asdict(dc)
            d["mode"] = dc.mode.value
            assert json.loads(json.dumps(d)) == g[f"dynamics.{cond}"], (name, cond)
    with pytest.raises(ValueError):
        C.get_preset("nope")
    with pytest.raises(ValueError):
        C.TrainConfig(mode="bogus")
    with pytest.raises(ValueError):
        C.TrainConfig(seq_len=1)
    with pytest.raises(ValueError):
        C.TrainConfig(conditioning="sideways")
