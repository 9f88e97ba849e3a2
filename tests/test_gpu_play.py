"""Device play sessions (paper_2510_27002_b200/play.py, the transport-free core of deskworld's
PlayService, server.py:55-135): protocol and error codes, PNG frames, and the KV-cached session
against stateless decode_frame calls on the same generator (the reference's semantics, which
re-run the whole clip every act)."""
import json
from pathlib import Path
import base64
import io

import numpy as np
import pytest
import torch

from oracle import rng as OR

pytestmark = pytest.mark.gpu
TOL = json.loads((Path(__file__).resolve().parent.parent / "fidelity_threshold.json").read_text())["parity"]

DKW = dict(model_dim=128, heads=2, ffn_dim=512, blocks=2, token_codes=256, action_latent_dim=32,
           patches_per_frame=256, max_frames=6)


def _episode(seed, n):
    return OR.stream(31, "episode", seed).integers(0, 256, size=(n, 64, 64, 3)).astype(np.uint8)


def _service(scale_logits=1.0, steps=4):
    from paper_2510_27002_b200.dynamics import ConditioningMode, DynamicsConfig, DynamicsModel
    from paper_2510_27002_b200.play import PlayService
    from paper_2510_27002_b200.tokenizer import TokenizerConfig, VideoTokenizer
    tok = VideoTokenizer(TokenizerConfig(model_dim=128, heads=2, ffn_dim=512, blocks=1, codes=256, latent_dim=32,
                                         patch=4, max_frames=8), seed=6)
    dyn = DynamicsModel(DynamicsConfig(**DKW, mode=ConditioningMode.GROUND_TRUTH), seed=7)
    if scale_logits != 1.0:
        dyn.params["to_logits.w"].data.mul_(scale_logits)
    return PlayService(tok, dyn, episode_fn=_episode, steps=steps), tok, dyn


def _png_frame(b64):
    from PIL import Image
    return np.asarray(Image.open(io.BytesIO(base64.b64decode(b64))).convert("RGB"))


def test_play_protocol_and_errors():
    from paper_2510_27002_b200.play import PlayService
    svc, tok, dyn = _service()
    assert svc.handle([1])["code"] == "bad_message"
    assert svc.handle({"type": "jump"})["code"] == "bad_type"
    assert svc.handle({"type": "act", "session": "nope", "action": 0})["code"] == "unknown_session"
    r = svc.handle({"type": "reset", "seed": 5})
    assert r["type"] == "frames" and r["step"] == 0 and len(r["png_base64"]) == 4
    sid = r["session"]
    assert sid == "s5-0"
    assert svc.handle({"type": "act", "session": sid})["code"] == "bad_action"
    assert svc.handle({"type": "act", "session": sid, "action": "x"})["code"] == "bad_action"
    assert svc.handle({"type": "act", "session": sid, "action": 7})["code"] == "action_out_of_range"
    a = svc.handle({"type": "act", "session": sid, "action": 3})
    assert a["type"] == "frames" and a["step"] == 1 and len(a["png_base64"]) == 1
    assert _png_frame(a["png_base64"][0]).shape == (64, 64, 3)
    # the reset frames are the tokenizer's reconstruction of the episode (server.py:104)
    shown = _png_frame(r["png_base64"][0])
    rec = svc._frames_u8(tok.encode_device(torch.as_tensor(_episode(5, 4)[None], device="cuda")))[0]
    np.testing.assert_array_equal(shown, rec)
    assert PlayService(tok, dyn).handle({"type": "reset"})["code"] == "no_environment"


def test_play_session_kv_cache_matches_stateless_decode():
    """Acts through the session's KV cache, including the window slide at max_frames (6), against
    the reference semantics: decode_frame over the whole (slid) clip on every act, same generator."""
    from paper_2510_27002_b200.play import N_CONDITIONING
    from paper_2510_27002_b200.rng import fold_key, stream
    from paper_2510_27002_b200.sampling import decode_frame_device
    svc, tok, dyn = _service(scale_logits=30.0)
    sid = svc.handle({"type": "reset", "seed": 2, "session": "p"})["session"]
    actions = [1, 4, 0, 6, 2]
    for a in actions:
        assert svc.handle({"type": "act", "session": sid, "action": a})["type"] == "frames"
    sess = svc.sessions[sid]
    assert sess.tokens.shape[1] == DKW["max_frames"]  # slid twice: 4 + 5 acts capped at 6

    # teacher-forced stateless replay with the reference's bookkeeping (server.py:108-130): before
    # every act the clip is the session's own (slid) token history, and decode_frame re-runs it all
    tokens = tok.encode_device(torch.as_tensor(_episode(2, N_CONDITIONING)[None], device="cuda"))
    null = dyn.params["null_action"].data.reshape(1, 1, -1)
    history = torch.zeros(1, N_CONDITIONING - 1, null.shape[-1], device="cuda") + null
    rng = stream(fold_key("p"), "play")
    table = dyn.params["gt_action_embed"].data
    assert len(sess.frames) == N_CONDITIONING + len(actions)
    for k, a in enumerate(actions):
        history = torch.cat([history, table[a].reshape(1, 1, -1)], dim=1)
        slid = tokens.shape[1] + 1 > DKW["max_frames"]
        if slid:
            tokens, history = tokens[:, 1:], history[:, 1:]
        ref = decode_frame_device(dyn, tokens, history, steps=4, temperature=1.0, rng=rng)[0]
        got = sess.generated[k]
        if k == 0:
            # prefill + decode: the same computation as decode_frame
            assert torch.equal(got, ref)
        else:
            # the session read K/V it appended through the single-frame path (a slide re-prefills):
            # equal to the full recompute within bf16 rounding, so only near-tie draws may differ
            assert float((got == ref).float().mean()) >= TOL["decode_token_agreement_peaked"], (k, float((got == ref).float().mean()))
        tokens = torch.cat([tokens, got[None, None]], dim=1)
    assert torch.equal(tokens, sess.tokens)
