"""ORACLE — CPU restatement of the deskworld hot path.  TEST INFRASTRUCTURE ONLY.

This package restates, from the reference source, the algorithms of the
Jasmine/Genie hot path so the B200 product can be checked against them:

  oracle.rng    splitmix64 / fold_key / numpy Philox4x64-10 stream layout,
                counter skip-ahead, sample_masks         (deskworld/rng.py, dynamics.py:52-62)
  oracle.model  nn ops, ST block/stack, tokenizer, LAM, dynamics logits/loss,
                VQ, MaskGIT sampler, rollout, AdamW/WSD    (deskworld/{nn,st,tokenizer,lam,
                                                            dynamics,optim}.py)

Floating-point parts are written with torch on the CPU (fp32 or fp64) so that
gradients come from torch.autograd; integer/bool parts (keys, Philox words,
masks, keep schedules) are exact numpy/pure-Python integer arithmetic.

Pinning: tests/test_oracle_golden.py checks this oracle against golden vectors
that tests/golden/make_golden.py produced by importing the UNMODIFIED reference
(/root/reference/pkg/src) in the build container: fold_key values, raw Philox
words, masks, VQ indices/losses, and the forward values AND every parameter
gradient of small tokenizer / LAM / dynamics models in float64, MaskGIT decode
and rollout outputs, and AdamW steps.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this package, and only as the checker.  The product
(paper_2510_27002_b200) never imports it.
"""
