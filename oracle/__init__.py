"""Plain, slow, obviously-correct CPU oracle for the DD-PPO learner step.

TEST INFRASTRUCTURE ONLY.  Nothing on the product path may import, call,
link or execute anything under ``oracle/``; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may.  The oracle shares no code with the CUDA path
(``paper_1911_00357_b200/``) and imports nothing from it; the two meet only
in ``synth/`` (seeded input generators, none of the method's arithmetic).

Everything is NumPy float64 over the (fp32) inputs.  Citations use
``P:Lnn`` = /root/reference/PAPER.md line nn (section in parentheses) and
``S:Lnn`` = /root/reference/SPEC.md line nn.  Readings of silent/ambiguous
passages are the Z-ledger of SURVEY.md section 8(c), repeated in DESIGN.md.

Parity status per function (the pins live in tests/test_oracle_*.py):
  gae.gae                      pinned (tau=1 closed form, tau=0 = TD error,
                               O(T^2) brute force, single terminal step)
  advnorm.*                    pinned (moments of the normalised buffer,
                               N ranks == concatenation)
  ppo.loss_and_grad            pinned (ratio==1 identity, Eq.2 worked value,
                               uniform-logit entropy, finite differences,
                               torch.autograd fp64)
  optim.*                      pinned (SPEC allreduce example, first Adam step,
                               torch.optim.Adam / clip_grad_norm_)
  preempt.*                    pinned (closed form == independent tick
                               simulation, SPEC arithmetic examples)
  minibatch.*                  pinned (exact cover per epoch)
  nets.* / models.*            pinned (torch.nn fp64 modules + autograd,
                               finite differences, zero-parameter identities)
  learner.learner_step         composition of the above; pinned by the
                               N=2-identical-buffers == N=1 identity and the
                               equal-weighting identity
"""
