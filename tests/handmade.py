"""Hand-built problem descriptions for the pin tests (raw inputs only)."""
import numpy as np

from workloads.synth import Problem


def hand_problem(model, n_req, mu, var, slo, *, Q=1, D=1, M=None, theta=1000.0,
                 prefill=0.5, eps=1.2, dtok=0.025, max_out=2048.0, swap=20.0,
                 q_device=None, q_resident=None, backlog_mean=None, backlog_var=None,
                 len_tables=None, dist=None):
    model = np.asarray(model, np.int32)
    G = len(model)
    M = int(model.max()) + 1 if M is None else M

    def full(x, shape):
        a = np.asarray(x, np.float64)
        return np.broadcast_to(a, shape).copy()

    sw = full(swap, (D, M, M))
    for d in range(D):
        np.fill_diagonal(sw[d], 0.0)
    return Problem(
        name="hand", model=model, n_req=np.asarray(n_req, np.int32) * np.ones(G, np.int32),
        slo=full(slo, (G,)), mu=full(mu, (G,)), var=full(var, (G,)),
        dist=np.full(G, -1, np.int32) if dist is None else np.asarray(dist, np.int32),
        q_device=np.zeros(Q, np.int32) if q_device is None else np.asarray(q_device, np.int32),
        q_resident=np.zeros(Q, np.int32) if q_resident is None else np.asarray(q_resident, np.int32),
        q_backlog_mean=np.zeros(Q) if backlog_mean is None else full(backlog_mean, (Q,)),
        q_backlog_var=np.zeros(Q) if backlog_var is None else full(backlog_var, (Q,)),
        theta=full(theta, (D, M)), prefill=full(prefill, (D, M)), eps=full(eps, (D, M)),
        dtok=full(dtok, (D, M)), max_out=full(max_out, (D, M)), swap=sw,
        len_tables=len_tables,
    )


def rank_of(order):
    """Lexicographic rank of a permutation (for readable test assertions)."""
    order = list(order)
    n = len(order)
    rank = 0
    avail = sorted(order)
    fact = [1] * (n + 1)
    for k in range(1, n + 1):
        fact[k] = fact[k - 1] * k
    for pos, x in enumerate(order):
        k = avail.index(x)
        rank += k * fact[n - 1 - pos]
        avail.pop(k)
    return rank
