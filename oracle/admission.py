"""Oracle of the saturation-bounded admission (NEXT-4) -- TEST INFRASTRUCTURE ONLY.

Plain-Python transcription of Algorithm 1 (App. A) and of the Eq. 2 cost
 with the functional forms of reading R18 (SPEC.md's standard terms):
    C_pfx(n)   = n f_tok + 2 n^2 HL
    C_sfx(S,P) = S f_tok + 2 S^2 HL + 4 S P HL
Shares no code with paper_2605_02960_b200."""


def c_pfx(n, f_tok, hl):
    return n * f_tok + 2.0 * n * n * hl


def c_sfx(S, P, f_tok, hl):
    return S * f_tok + 2.0 * S * S * hl + 4.0 * S * P * hl


def cost_delta(P, M, S, f_tok, hl):
    """Eq. 2: Delta_r = C_pfx(P_r - M_r) + C_sfx(S_r, P_r)."""
    assert 0 <= M <= P and S >= 0
    return c_pfx(P - M, f_tok, hl) + c_sfx(S, P, f_tok, hl)


def schedule_round(tables, loads, T, block_size, f_tok, hl, chains, prefix_len, suffix_len, reset=True):
    """One round of Algorithm 1.  tables[i] = set of block hashes (committed U pending) of GPU i,
    loads[i] = L_i; both updated in place.  Returns (gpu per request or -1, delta per request)."""
    N = len(loads)
    if reset:
        for i in range(N):
            loads[i] = 0.0                       # L_i <- 0
    active = [loads[i] < T for i in range(N)]    # A <- {i : L_i < T}
    gpus, deltas = [], []
    for chain, P, S in zip(chains, prefix_len, suffix_len):   # in arrival order
        if not any(active):                     # if A = {} then break (request stays queued)
            gpus.append(-1)
            deltas.append(0.0)
            continue
        best, best_m = None, -1
        for i in range(N):
            if not active[i]:
                continue
            m = 0                                # m_i <- BlockMatch(K_i, r)
            while m < len(chain) and chain[m] in tables[i]:
                m += 1
            # i* = argmax m_i; ties -> argmin L_i; then lowest index
            if m > best_m or (m == best_m and loads[i] < loads[best]):
                best, best_m = i, m
        d = cost_delta(P, min(best_m * block_size, P), S, f_tok, hl)
        loads[best] += d                         # L_{i*} <- L_{i*} + Delta
        tables[best].update(chain)               # its blocks are now (pending) on i*
        if loads[best] >= T:                     # if L_{i*} >= T then A <- A \\ {i*}
            active[best] = False
        gpus.append(best)
        deltas.append(d)
    return gpus, deltas
