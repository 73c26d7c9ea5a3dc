"""PPIEM scan oracle -- TEST INFRASTRUCTURE ONLY (tests/ may import it; the product path never
does).  Plain Python over the C oracle scorer (oracle_score.c), following DESIGN.md reading A23:

Algorithm PPIEM, steps A3-A6:
  A3  each (position j, orientation k) starts at centre + s_start u_j and approaches the centre
      along the line by sphere tracing on the pose's minimum distance d:
          d = +inf:           s <- s - (D_cap - sigma)
          d - sigma <= tol:   contact (status 0)
          otherwise:          s <- s - (d - sigma) * 0.999
      status 1: an atom left the box (NaN); 2: clash at s_start; 3: s < 0; 4: max_iter reached.
  A4/A5 the energy at the final position of every (j, k).
  A6  local minima on the grid periodic in both indices (ties toward the smaller index).
Shares no code with the library; the scorer is the oracle's O1-O8."""
from __future__ import annotations

import numpy as np

from . import rs_oracle


def poses_at(centre, dirs, quats, s):
    m_P, m_L = s.shape
    P = np.empty((m_P, m_L, 7))
    P[:, :, :4] = quats[None, :, :]
    for a in range(3):
        P[:, :, 4 + a] = centre[a] + s * dirs[:, None, a]
    return P.reshape(-1, 7)


def scan(tables, X, qM, Y, zL, centre, dirs, quats, s_start, sigma, dcap, tol=1e-3, max_iter=64):
    centre = np.asarray(centre, float)
    m_P, m_L = dirs.shape[0], quats.shape[0]
    s = np.full((m_P, m_L), float(s_start))
    status = np.full((m_P, m_L), -1, dtype=np.int32)
    E = np.full((m_P, m_L), np.nan)
    moved = True
    it = 0
    while it < max_iter and moved:
        Ep, dp, _ = rs_oracle.score_poses(tables, X, qM, Y, zL, poses_at(centre, dirs, quats, s), dcap)
        Ep = Ep.reshape(m_P, m_L)
        dp = dp.reshape(m_P, m_L)
        moved = False
        for j in range(m_P):
            for k in range(m_L):
                if status[j, k] != -1:
                    continue
                E[j, k] = Ep[j, k]
                d = dp[j, k]
                if np.isnan(d):
                    status[j, k] = 1
                    continue
                if np.isinf(d):
                    sn = s[j, k] - (dcap - sigma)
                else:
                    delta = d - sigma
                    if delta < 0.0:
                        # later only rounding puts d below sigma: contact (A23)
                        status[j, k] = 2 if it == 0 else 0
                        continue
                    if delta <= tol:
                        status[j, k] = 0
                        continue
                    sn = s[j, k] - delta * 0.999
                if sn < 0.0:
                    status[j, k] = 3
                    continue
                s[j, k] = sn
                moved = True
        it += 1
    if moved:
        Ep, _, _ = rs_oracle.score_poses(tables, X, qM, Y, zL, poses_at(centre, dirs, quats, s), dcap)
        Ep = Ep.reshape(m_P, m_L)
        act = status == -1
        E[act] = Ep[act]
    status[status == -1] = 4
    E[(status != 0) & (status != 4)] = np.nan
    return E, s, status


def landscape_minima(E, top_k):
    """A6: flat indices of strict local minima (periodic 8-neighbourhood, ties toward the
    lexicographically smaller index, NaN skipped), sorted by energy then index."""
    m_P, m_L = E.shape
    mins = []
    for j in range(m_P):
        for k in range(m_L):
            e = E[j, k]
            if np.isnan(e):
                continue
            ok = True
            for dj in (-1, 0, 1):
                for dk in (-1, 0, 1):
                    jj, kk = (j + dj) % m_P, (k + dk) % m_L
                    if (jj, kk) == (j, k):
                        continue
                    f = E[jj, kk]
                    if np.isnan(f):
                        continue
                    if f < e or (f == e and (jj, kk) < (j, k)):
                        ok = False
            if ok:
                mins.append(j * m_L + k)
    mins.sort(key=lambda i: (E.flat[i], i))
    return np.array(mins[:top_k], dtype=np.int32)
