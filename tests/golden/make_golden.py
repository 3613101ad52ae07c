"""Generate golden fixtures by running the REFERENCE itself (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Imports ``triad`` (the reference, read-only at /root/reference) and records
its own outputs -- ``group_loss`` / ``combine_reports`` (algorithms.py:351-379),
``loss_sft`` (256-274), ``loss_dpo`` (277-315), ``regularizer_g`` (193-217),
``policy.logprob`` per-token values (policy.py:194-212), the scored states
(policy.py:181-191) and ``ExperienceBuffer.sample_batch(group_by_task=True)``
group indexing (buffer.py:215-267) -- into small ``.npz`` fixtures that travel
with the repo.  The GPU box never sees /root/reference; tests there only read
these files.
"""

from __future__ import annotations

import math
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from triad import algorithms as A  # noqa: E402
from triad import policy as P  # noqa: E402
from triad.buffer import ExperienceBuffer  # noqa: E402
from triad.orchestrator import Trainer  # noqa: E402
from triad.records import Experience, ExperienceState, TaskGroup  # noqa: E402

OUT = Path(__file__).resolve().parent


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float64 -> bf16 (RNE) -> float64, so GPU and reference see identical values."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def make_experience(rng, vocab, task_key, n_prompt, n_turns, max_span, behavior, multi_turn):
    """Single- or multi-turn experience with interior mask-false spans
    (workflows.py:128-183 layout: role markers and env text are mask-false)."""
    prompt = [int(x) for x in rng.integers(-3, vocab.size, size=n_prompt)]
    tokens = list(prompt)
    mask = [False] * len(prompt)
    for turn in range(n_turns):
        span = int(rng.integers(1, max_span + 1))
        gen = [int(x) for x in rng.integers(0, vocab.size, size=span)]
        tokens += gen
        mask += [True] * span
        if multi_turn and turn + 1 < n_turns:
            env = [int(x) for x in rng.integers(-3, vocab.size, size=int(rng.integers(1, 4)))]
            tokens += env
            mask += [False] * len(env)
    resp = P.Response(tokens=tokens, prompt_length=len(prompt),
                      logprobs=[0.0] * sum(mask), action_mask=mask)
    _, per = P.logprob(behavior, prompt, resp)
    lps = [per[i] for i in range(len(tokens)) if mask[i]]
    return Experience(task_key=task_key, tokens=tokens, prompt_length=len(prompt),
                      action_mask=mask, logprobs=lps, reward=float(rng.uniform(-1, 1)),
                      model_version=0)


def table(rng, S, V, scale, bf16):
    t = rng.normal(0.0, scale, size=(S, V))
    return bf16_round(t) if bf16 else t


def flatten_groups(groups):
    toks, tok_off, plen, masks, lps, lp_off, rew, gsize, refs = [], [0], [], [], [], [0], [], [], []
    for g in groups:
        gsize.append(g.size)
        refs += list(g.ref_logprobs)
        for e in g.experiences:
            toks += e.tokens
            masks += [1 if m else 0 for m in e.action_mask]
            tok_off.append(len(toks))
            plen.append(e.prompt_length)
            lps += e.logprobs
            lp_off.append(len(lps))
            rew.append(float(e.reward))
    return dict(tokens=np.array(toks, np.int64), tok_off=np.array(tok_off, np.int64),
                prompt_len=np.array(plen, np.int64), mask=np.array(masks, np.int8),
                logprobs=np.array(lps), lp_off=np.array(lp_off, np.int64),
                reward=np.array(rew), group_size=np.array(gsize, np.int64),
                ref_logprobs=np.array(refs))


def states_of(groups, S):
    st, tg, lp_tok = [], [], []
    for g in groups:
        for e in g.experiences:
            key = P.sequence_key(e.tokens[: e.prompt_length])
            for _, s, t in P.scored_states(P.PolicyParams(np.zeros((S, 2)), 0, P.Vocabulary(2, 0)), key, e.tokens, e.action_mask):
                st.append(s)
                tg.append(t)
    return np.array(st, np.int64), np.array(tg, np.int64)


def per_token_lp(groups, params):
    out = []
    for g in groups:
        for e in g.experiences:
            _, per = P.logprob(params, e.tokens[: e.prompt_length],
                               P.Response(e.tokens, e.prompt_length, e.logprobs, e.action_mask))
            out += [per[i] for i in range(len(e.tokens)) if e.action_mask[i]]
    return np.array(out)


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print("wrote", name, {k: getattr(v, "shape", v) for k, v in arrays.items() if hasattr(v, "shape")})


def group_case(name, seed, V, S, n_groups, K, variant, tau, beta, scale=0.8, bf16=False,
               multi_turn=True, ref_params_mode=False):
    rng = np.random.default_rng(seed)
    vocab = P.Vocabulary(size=V, eos_token=V - 1)
    theta = table(rng, S, V, scale, bf16)
    anchor = table(rng, S, V, scale, bf16)
    behavior = P.PolicyParams(table(rng, S, V, scale * 0.5, bf16), 0, vocab)
    params = P.PolicyParams(theta, 0, vocab)
    anchor_p = P.PolicyParams(anchor, 0, vocab)
    groups = []
    for g in range(n_groups):
        exps = [make_experience(rng, vocab, 1000 + g, int(rng.integers(1, 4)),
                                int(rng.integers(1, 4)), 5, behavior, multi_turn)
                for _ in range(K)]
        # distinct per-group reward patterns incl. an all-equal group
        if g == 0 and n_groups > 2:
            for e in exps:
                e.reward = 0.5
        groups.append(TaskGroup(1000 + g, exps))
    cfg = A.AlgorithmConfig(variant, tau=tau, beta=beta)
    reps = [A.group_loss(g, params, cfg, sft_params=anchor_p) for g in groups]
    comb = A.combine_reports(reps)
    st, tg = states_of(groups, S)
    save(name, theta=theta, anchor=anchor, states=st, target=tg,
         lp_tok=per_token_lp(groups, params),
         loss=np.array(comb.loss), grad=comb.gradient.to_dense((S, V)),
         group_losses=np.array([r.loss for r in reps]),
         metric_names=np.array(sorted(comb.metrics)),
         metric_values=np.array([comb.metrics[k] for k in sorted(comb.metrics)]),
         variant=np.array(variant), tau=np.array(tau), beta=np.array(beta),
         **flatten_groups(groups))


def sft_case(name, seed, V, S, n):
    rng = np.random.default_rng(seed)
    vocab = P.Vocabulary(size=V, eos_token=V - 1)
    params = P.PolicyParams(table(rng, S, V, 0.8, False), 0, vocab)
    behavior = P.PolicyParams(table(rng, S, V, 0.3, False), 0, vocab)
    batch = [make_experience(rng, vocab, 7, int(rng.integers(1, 3)), int(rng.integers(1, 3)), 6,
                             behavior, True) for _ in range(n)]
    rep = A.loss_sft(batch, params)
    grp = [TaskGroup(7, batch)]
    st, tg = states_of(grp, S)
    save(name, theta=params.logits, states=st, target=tg, loss=np.array(rep.loss),
         grad=rep.gradient.to_dense((S, V)),
         metric_names=np.array(sorted(rep.metrics)),
         metric_values=np.array([rep.metrics[k] for k in sorted(rep.metrics)]),
         **flatten_groups(grp))


def dpo_case(name, seed, V, S, n_pairs, dpo_beta):
    rng = np.random.default_rng(seed)
    vocab = P.Vocabulary(size=V, eos_token=V - 1)
    params = P.PolicyParams(table(rng, S, V, 0.8, False), 0, vocab)
    ref = P.PolicyParams(table(rng, S, V, 0.8, False), 0, vocab)
    sampler = P.PolicyParams(table(rng, S, V, 0.2, False), 0, vocab)
    pairs = []
    for i in range(n_pairs):
        c = make_experience(rng, vocab, 3, 2, 1, 5, sampler, False)
        r = make_experience(rng, vocab, 3, 2, 1, 5, sampler, False)
        r.tokens[: r.prompt_length] = c.tokens[: c.prompt_length]
        r = Experience(task_key=3, tokens=c.tokens[: c.prompt_length] + r.tokens[r.prompt_length:],
                       prompt_length=c.prompt_length, action_mask=r.action_mask,
                       logprobs=r.logprobs, reward=0.0, model_version=0)
        pairs.append((c, r))
    rep = A.loss_dpo(pairs, params, ref, dpo_beta)
    grps = [TaskGroup(3, [c, r]) for c, r in pairs]
    ref_seq = [A.experience_logprob(ref, e) for c, r in pairs for e in (c, r)]
    st, tg = states_of(grps, S)
    save(name, theta=params.logits, anchor=ref.logits, states=st, target=tg,
         loss=np.array(rep.loss), grad=rep.gradient.to_dense((S, V)),
         ref_seq_lp=np.array(ref_seq), dpo_beta=np.array(dpo_beta),
         metric_names=np.array(sorted(rep.metrics)),
         metric_values=np.array([rep.metrics[k] for k in sorted(rep.metrics)]),
         **flatten_groups(grps))


def regularizer_case(name, seed, V, S, K):
    rng = np.random.default_rng(seed)
    vocab = P.Vocabulary(size=V, eos_token=V - 1)
    params = P.PolicyParams(table(rng, S, V, 0.8, False), 0, vocab)
    anchor = P.PolicyParams(table(rng, S, V, 0.8, False), 0, vocab)
    behavior = P.PolicyParams(table(rng, S, V, 0.3, False), 0, vocab)
    exps = [make_experience(rng, vocab, 5, 2, 2, 4, behavior, True) for _ in range(K)]
    grp = [TaskGroup(5, exps)]
    value, grad = A.regularizer_g(params, anchor, grp[0])
    st, tg = states_of(grp, S)
    save(name, theta=params.logits, anchor=anchor.logits, states=st, target=tg,
         value=np.array(value), grad=grad.to_dense((S, V)), **flatten_groups(grp))


def buffer_case(name, seed, n_exp, n_tasks, group_size, n_take, policy):
    """ExperienceBuffer.sample_batch(group_by_task=True) group indexing."""
    rng = np.random.default_rng(seed)
    tasks = rng.integers(0, n_tasks, size=n_exp)
    prio = np.round(rng.uniform(0, 3, size=n_exp), 1)
    ready = rng.uniform(size=n_exp) < 0.85
    with tempfile.TemporaryDirectory() as d:
        buf = ExperienceBuffer(Path(d) / "buf.jsonl")
        ids = []
        for i in range(n_exp):
            e = Experience(task_key=int(tasks[i]), tokens=[1, 2], prompt_length=1,
                           action_mask=[False, True], logprobs=[-0.5],
                           reward=0.0 if ready[i] else None, model_version=0,
                           state=ExperienceState.READY if ready[i] else ExperienceState.PENDING_REWARD,
                           priority=float(prio[i]))
            ids.append(buf.put(e))
        res = buf.sample_batch(n_take, policy=policy, group_by_task=True, group_size=group_size)
        pos = {sid: i for i, sid in enumerate(ids)}
        out = [[pos[e.sample_id] for e in g.experiences] for g in res.groups]
    save(name, tasks=tasks, priority=prio, ready=ready, group_size=np.array(group_size),
         n_take=np.array(n_take), policy=np.array(policy),
         groups=np.array(out, np.int64).reshape(-1, group_size), short=np.array(res.short))


def trainer_case(name, seed, V, S, n_groups, K, variant, tau, beta, steps, lr, sft_n=0,
                 dpo_pairs=0):
    """The reference's own Trainer (orchestrator.py:288-322): `steps` x
    step_groups (+ a step_sft / step_dpo at the end), recording every step's
    loss and metrics and the final table and version."""
    rng = np.random.default_rng(seed)
    vocab = P.Vocabulary(size=V, eos_token=V - 1)
    behavior = P.PolicyParams(table(rng, S, V, 0.4, False), 0, vocab)
    params = P.PolicyParams(table(rng, S, V, 0.8, False), 0, vocab)
    groups = []
    for g in range(n_groups):
        exps = [make_experience(rng, vocab, 1000 + g, int(rng.integers(1, 4)),
                                int(rng.integers(1, 4)), 5, behavior, True) for _ in range(K)]
        groups.append(TaskGroup(1000 + g, exps))
    tr = Trainer(params, A.AlgorithmConfig(variant, tau=tau, beta=beta, learning_rate=lr))
    losses, metrics = [], []
    for _ in range(steps):
        rep = tr.step_groups(groups)
        losses.append(rep.loss)
        metrics.append([rep.metrics[k] for k in sorted(rep.metrics)])
    extra = {}
    if sft_n:
        batch = [make_experience(rng, vocab, 7, 2, 2, 5, behavior, True) for _ in range(sft_n)]
        losses.append(tr.step_sft(batch).loss)
        extra.update(sft=flatten_groups([TaskGroup(7, batch)]))
    if dpo_pairs:
        pairs = []
        for _ in range(dpo_pairs):
            c = make_experience(rng, vocab, 3, 2, 1, 5, behavior, False)
            r = make_experience(rng, vocab, 3, 2, 1, 5, behavior, False)
            r = Experience(task_key=3, tokens=c.tokens[: c.prompt_length] + r.tokens[r.prompt_length:],
                           prompt_length=c.prompt_length, action_mask=r.action_mask,
                           logprobs=r.logprobs, reward=0.0, model_version=0)
            pairs.append((c, r))
        losses.append(tr.step_dpo(pairs).loss)
        extra.update(dpo=flatten_groups([TaskGroup(3, [c, r]) for c, r in pairs]))
    flat = {f"{k2}_{k}": v for k2, d in extra.items() for k, v in d.items()}
    save(name, theta=params.logits, final=tr.params.logits, version=np.array(tr.params.version),
         losses=np.array(losses), metric_names=np.array(sorted(rep.metrics)),
         metric_values=np.array(metrics), variant=np.array(variant), tau=np.array(tau),
         beta=np.array(beta), lr=np.array(lr), steps=np.array(steps), **flat,
         **flatten_groups(groups))


def known_answers():
    """Frozen values from the reference tests (test_algorithms.py:109-188)."""
    vals = {
        "tau_log_zhat_ln5": A.tau_log_zhat([0.0, math.log(9.0)], 1.0),
        "tau_log_zhat_1000": A.tau_log_zhat([1000.0, 1000.0], 1.0),
    }
    save("known_answers", names=np.array(sorted(vals)),
         values=np.array([vals[k] for k in sorted(vals)]))


def main():
    group_case("simple_tau05", 101, V=64, S=32, n_groups=3, K=4, variant="OPMD_SIMPLE", tau=0.5, beta=0.0)
    group_case("simple_tau0", 102, V=64, S=32, n_groups=4, K=4, variant="OPMD_SIMPLE", tau=0.0, beta=0.0)
    group_case("simple_anchor", 103, V=48, S=24, n_groups=2, K=3, variant="OPMD_SIMPLE", tau=0.4, beta=0.9)
    group_case("kimi", 104, V=64, S=32, n_groups=3, K=4, variant="OPMD_KIMI", tau=0.7, beta=0.0)
    group_case("pairwise", 105, V=64, S=32, n_groups=3, K=4, variant="OPMD_PAIRWISE", tau=1.3, beta=0.0)
    group_case("simple_bf16_v512", 106, V=512, S=64, n_groups=3, K=8, variant="OPMD_SIMPLE", tau=1.0,
               beta=0.0, scale=2.0, bf16=True)
    group_case("kimi_bf16_v512", 107, V=512, S=64, n_groups=2, K=8, variant="OPMD_KIMI", tau=1.0,
               beta=0.0, scale=2.0, bf16=True)
    group_case("simple_v4_uniform", 108, V=4, S=6, n_groups=2, K=3, variant="OPMD_SIMPLE", tau=0.0,
               beta=0.0, scale=1e-300)
    sft_case("sft", 201, V=32, S=16, n=5)
    dpo_case("dpo", 301, V=32, S=16, n_pairs=4, dpo_beta=0.3)
    regularizer_case("regularizer_g", 401, V=40, S=20, K=3)
    buffer_case("buffer_fifo", 501, n_exp=60, n_tasks=5, group_size=4, n_take=6, policy="FIFO")
    buffer_case("buffer_priority", 502, n_exp=60, n_tasks=4, group_size=3, n_take=50, policy="PRIORITY")
    known_answers()
    trainer_case("trainer_simple_anchor", 601, V=48, S=24, n_groups=2, K=3, variant="OPMD_SIMPLE",
                 tau=0.5, beta=0.4, steps=3, lr=0.2, sft_n=3, dpo_pairs=2)
    trainer_case("trainer_kimi", 602, V=64, S=32, n_groups=2, K=4, variant="OPMD_KIMI", tau=0.8,
                 beta=0.0, steps=3, lr=0.1)


if __name__ == "__main__":
    main()
