"""Mutation check of the oracle's pins (tests/, -m "not gpu"): each mutation below is a plausible
mistake in oracle/squint_oracle.py; applied to a scratch copy of the repo, at least one oracle test
must fail.  ``python tools/oracle_mutations.py`` prints CAUGHT / SURVIVED per mutation."""
import os, shutil, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
muts = {
 "done_mask": ('    not_done = 1.0 - done.astype(np.float64)                                          # Q22',
               '    not_done = np.ones(len(done))'),
 "act_proj": ('    zp, _ = projection_fwd(actor, "actor", h, hp.ln_eps)\n    out, _ = mlp_fwd(actor, "actor", _head_input(zp, proprio',
              '    zp, _ = projection_fwd(critic, "critic", h, hp.ln_eps)\n    out, _ = mlp_fwd(actor, "actor", _head_input(zp, proprio'),
 "entropy_sign": ('float(-logp.mean()), gnorm', 'float(logp.mean()), gnorm'),
 "alpha0_actor": ('st["actor"], h, s, at, logp, caches, alpha1, scale)', 'st["actor"], h, s, at, logp, caches, alpha0, scale)'),
 "pre_step_theta": ('    Lpi, gpi, qmean = actor_loss_and_grads(d, hp, st["critic"],', '    Lpi, gpi, qmean = actor_loss_and_grads(d, hp, _pre_critic,'),
 "shift_swap": ('O = shift_images(R["obs"][idx], shift[:, 0], shift[:, 1], p)', 'O = shift_images(R["obs"][idx], shift[:, 1], shift[:, 0], p)'),
 "shift_obs_next": ('O = shift_images(R["obs"][idx], shift[:, 0], shift[:, 1], p)', 'O = shift_images(R["obs"][idx], shift[:, 2], shift[:, 3], p)'),
 "ln_eps_outside": ('    rstd = 1.0 / np.sqrt(var + eps)', '    rstd = 1.0 / (np.sqrt(var) + eps)'),
 "ln_bwd_drop_term": ('dx = rstd * (dxh - dxh.mean(axis=-1, keepdims=True) - xh * (dxh * xh).mean(axis=-1, keepdims=True))',
                      'dx = rstd * (dxh - dxh.mean(axis=-1, keepdims=True))'),
 "adam_bias_t": ('    mhat = m / (1.0 - b1 ** t)', '    mhat = m / (1.0 - b1 ** (t + 1))'),
 "polyak_swap": ('    return (1.0 - tau) * target + tau * online', '    return tau * target + (1.0 - tau) * online'),
 "squash_sign": ('- 0.5 * LOG_2PI - np.log(1.0 - a * a + SQUASH_EPS)).sum(axis=1)', '- 0.5 * LOG_2PI + np.log(1.0 - a * a + SQUASH_EPS)).sum(axis=1)'),
 "proj_weights_swap": ('                m[b, lo] += p[b, j] * (hi - bj)\n                m[b, hi] += p[b, j] * (bj - lo)',
                       '                m[b, lo] += p[b, j] * (bj - lo)\n                m[b, hi] += p[b, j] * (hi - bj)'),
 "proj_gamma_missing": ('            g = r[b] + not_done[b] * gamma * (z[j] - shift[b])', '            g = r[b] + not_done[b] * (z[j] - shift[b])'),
 "proj_shift_sign": ('            g = r[b] + not_done[b] * gamma * (z[j] - shift[b])', '            g = r[b] + not_done[b] * gamma * (z[j] + shift[b])'),
 "rhe_floor": ('    return np.rint(s / float(factor * factor)).astype(np.uint8)', '    return np.floor(s / float(factor * factor)).astype(np.uint8)'),
 "tg_bwd_tanh_deriv": ('    dl = dlog_std * 0.5 * (hi - lo) * (1.0 - tl * tl)', '    dl = dlog_std * 0.5 * (hi - lo)'),
}
src = open(os.path.join(ROOT, "oracle", "squint_oracle.py")).read()
for name, (a, b) in muts.items():
    d = os.path.join(tempfile.gettempdir(), "squint_mut", name)
    if os.path.exists(d): shutil.rmtree(d)
    shutil.copytree(ROOT, d, ignore=shutil.ignore_patterns(".git", "gpurun_out", "scratch", "*.so", "build_obj"))
    assert src.count(a) == 1, name
    s = src.replace(a, b)
    if name == "pre_step_theta":
        s = s.replace('    # Lines 14-15: critic + encoder step.\n', '    # Lines 14-15: critic + encoder step.\n    _pre_critic = copy.deepcopy(st["critic"])\n')
        s = s.replace("def _update_one(d, hp, R, idx, shift, eps, st):", "def _update_one(d, hp, R, idx, shift, eps, st):\n    import copy")
    open(f"{d}/oracle/squint_oracle.py", "w").write(s)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider",
                        "tests/test_oracle_closed_forms.py", "tests/test_oracle_update.py", "tests/test_oracle_distributional.py",
                        "tests/test_oracle_layers.py", "tests/test_oracle_insert_shift.py"], cwd=d, capture_output=True, text=True)
    last = [l for l in r.stdout.splitlines() if "passed" in l or "failed" in l]
    print(name, "CAUGHT" if r.returncode != 0 else "SURVIVED", last[-1] if last else r.stdout[-300:])
