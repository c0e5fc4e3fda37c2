"""Error paths of the C ABI on the GPU (include/ddppo.h "Errors"): a non-finite value inside the
learner step is reported by ddppo_check as DDPPO_ERR_NUMERICAL and the parameter
update it would have produced is skipped; mismatched advantage-normalisation flags are a config
error."""
import numpy as np
import pytest
import torch

import paper_1911_00357_b200 as dd
import synth
from paper_1911_00357_b200.learner import Learner

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = dd.Context(0, 1, device=0)
    yield c
    c.close()


def _learner(ctx, arch="gps", **kw):
    c = synth.CONFIGS[arch]
    desc = dd.model_desc(arch)
    lay = dd.param_layout(desc)
    P = dd.param_count(desc)
    p0 = synth.init_params([(off, int(np.prod(s)), fan) for _, off, s, fan in lay], P, 3)
    lrn = Learner(ctx, arch, c["E"], 16, c["epochs"], c["minibatches"], params=p0, **kw)
    ro = synth.rollout(c["E"], 16, 3)
    return lrn, ro, synth.perms(3, 0, c["epochs"], c["E"]), p0


@pytest.mark.parametrize("where", ["rew", "val", "h0"])
def test_nan_reports_numerical_and_skips_update(ctx, where):
    lrn, ro, pm, p0 = _learner(ctx, normalize_adv=True)
    ro = dict(ro)
    ro[where] = ro[where].copy()
    ro[where][1, 3] = np.nan
    lrn.load_rollout(ro, pm)
    lrn.step()
    with pytest.raises(dd.DdppoError) as e:
        ctx.check()
    assert e.value.code == 2 and "non-finite" in str(e.value)
    prm = lrn.params.cpu().numpy()
    assert np.all(np.isfinite(prm))  # the non-finite update was never applied
    if where != "h0":  # NaN advantages reach every minibatch through the global statistics: no update at all
        assert np.array_equal(prm, p0)
    # the flag is cleared by the check: a clean rollout steps normally again
    lrn.load_rollout(synth.rollout(lrn.E, 16, 4), pm)
    lrn.step()
    ctx.check()
    assert not np.array_equal(lrn.params.cpu().numpy(), p0)


def test_mismatched_normalisation_flags_rejected(ctx):
    lrn, ro, pm, _ = _learner(ctx, normalize_adv=True)
    lrn.load_rollout(ro, pm)
    lrn.cfg.loss.normalize_adv = 0
    with pytest.raises(dd.DdppoError) as e:
        lrn.step()
    assert e.value.code == 1 and "agree" in str(e.value)
