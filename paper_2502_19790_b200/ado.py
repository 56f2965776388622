"""ADO (stage 3) behind the reference's API: ``per_domain_loss``,
``fit_power_law``, ``AdoState``, ``AdoSource`` (``ado.py:29-409``,
``client.py:582-598``).

Host objects keep the reference's state shape (tracks, history, fit_steps,
state_dict); the arithmetic runs on the device: the per-token segmented
reduction (``mx_domain_loss``), the batched power-law refit (one CTA per
domain, ``mx_fit_power_law``) and the pi / floor / temporal-average update
(``mx_ado_pi``, ``mx_ado_credit``), with mu, credit, pi and pi_bar resident in
HBM between chunks.
"""

from __future__ import annotations

import ctypes as C
import logging
import math
from dataclasses import dataclass, field
from typing import Mapping

import numpy as np

from . import _lib
from .errors import DataReadError, FeedbackError, MixtureError
from .mixtures import MixtureKey, MixtureSource, MixtureSpec, sorted_keys

logger = logging.getLogger(__name__)

_GEOM = None


def _geom(device):
    global _GEOM
    import torch

    if _GEOM is None or _GEOM.device != device:
        # the grid constant of fit_power_law (ado.py:143): numpy.geomspace(1e-6, 1, 49)
        _GEOM = torch.from_numpy(np.geomspace(1e-6, 1.0, 49)).to(device)
    return _GEOM


@dataclass
class AdoConfig:
    """Tuning knobs (``ado.py:29-70``)."""

    fit_start_step: int = 1000
    refit_every: int = 1000
    subsample_every: int = 10
    discard_first: int = 500
    p_min: float | None = None
    smoothing: float = 0.5
    credit_rate: float = 0.1
    samples_per_step: int = 1

    def __post_init__(self):
        if not (0 <= self.smoothing < 1):
            raise MixtureError("smoothing must lie in [0, 1)")
        if not (0 < self.credit_rate <= 1):
            raise MixtureError("credit_rate must lie in (0, 1]")
        if min(self.fit_start_step, self.refit_every, self.subsample_every) < 1:
            raise MixtureError("schedule parameters must be positive")

    def resolved_p_min(self, num_domains: int) -> float:
        p = 0.1 / num_domains if self.p_min is None else self.p_min
        if p * num_domains >= 1:
            raise MixtureError(f"p_min {p} too large for {num_domains} domains")
        return p

    def to_json(self) -> dict:
        return {k: getattr(self, k) for k in (
            "fit_start_step", "refit_every", "subsample_every", "discard_first",
            "p_min", "smoothing", "credit_rate", "samples_per_step")}

    @staticmethod
    def from_json(data: Mapping) -> "AdoConfig":
        return AdoConfig(**dict(data))


@dataclass(frozen=True)
class DomainLaw:
    epsilon: float
    beta: float
    alpha: float
    fallback: bool = False

    def predict(self, n: float) -> float:
        return self.epsilon + self.beta * n ** -self.alpha


def learning_speed(law: DomainLaw, n: float) -> float:
    if n < 1:
        raise ValueError("learning_speed requires n >= 1")
    return law.alpha * law.beta * n ** -(law.alpha + 1.0)


def fit_power_laws(histories: list[list[tuple[float, float]]], device="cuda") -> list[DomainLaw]:
    """Batched ``fit_power_law`` on the device: one CTA per history."""
    import torch

    for h in histories:
        if len(h) < 8:
            raise MixtureError("need at least 8 points to fit a power law")
    ns = np.concatenate([np.array([p[0] for p in h], dtype=np.float64) for h in histories])
    ls = np.concatenate([np.array([p[1] for p in h], dtype=np.float64) for h in histories])
    if np.any(ns < 1) or np.any(~np.isfinite(ls)):
        raise MixtureError("history points need n >= 1 and finite losses")
    off = np.zeros(len(histories) + 1, dtype=np.int64)
    np.cumsum([len(h) for h in histories], out=off[1:])
    dev = torch.device(device)
    t_off = torch.from_numpy(off).to(dev)
    t_n = torch.from_numpy(ns).to(dev)
    t_l = torch.from_numpy(ls).to(dev)
    out = torch.empty((len(histories), 4), dtype=torch.float64, device=dev)
    L = _lib.lib()
    _lib.check(L.mx_fit_power_law(len(histories), t_off.data_ptr(), t_n.data_ptr(), t_l.data_ptr(),
                                  _geom(dev).data_ptr(), out.data_ptr(), C.c_void_p(_lib.stream_ptr())))
    res = out.cpu().numpy()
    return [DomainLaw(float(e), float(b), float(a), bool(f)) for e, b, a, f in res]


def fit_power_law(history: list[tuple[float, float]]) -> DomainLaw:
    return fit_power_laws([list(history)])[0]


def per_domain_loss(token_losses, tags, domains=None, stream=None) -> dict:
    """``{tag: (loss sum f64, token count)}`` (``client.py:582-598``).

    ``token_losses``: f32 CUDA tensor (or any sequence). ``tags``: int32 CUDA
    tensor of domain indices into ``domains``, or a sequence of hashable tags
    (MixtureKeys) that is interned on the host first.
    """
    import torch

    if len(token_losses) != len(tags):
        raise DataReadError(f"{len(token_losses)} losses for {len(tags)} tags")
    dev = torch.device("cuda")
    if torch.is_tensor(tags):
        if domains is None:
            raise ValueError("integer tag tensors need the `domains` list")
        tag_t = tags.to(device=dev, dtype=torch.int32).contiguous()
        keys = list(domains)
    else:
        keys, index, idx = [], {}, []
        for t in tags:
            i = index.get(t)
            if i is None:
                i = index[t] = len(keys)
                keys.append(t)
            idx.append(i)
        tag_t = torch.tensor(idx, dtype=torch.int32, device=dev)
    loss_t = torch.as_tensor(token_losses, dtype=torch.float32, device=dev).contiguous()
    sums, counts = domain_loss_device(loss_t, tag_t, len(keys) or 1, stream)
    s, c = sums.cpu().tolist(), counts.cpu().tolist()
    return {k: (s[i], int(c[i])) for i, k in enumerate(keys) if c[i] > 0}


def domain_loss_device(losses, tags, n_domains: int, stream=None):
    """Device (sums f64[K], counts i64[K]) of one rank's tokens (no host sync
    beyond the error check)."""
    import torch

    sums = torch.empty(n_domains, dtype=torch.float64, device=losses.device)
    counts = torch.empty(n_domains, dtype=torch.int64, device=losses.device)
    _lib.check(_lib.lib().mx_domain_loss(losses.data_ptr(), tags.data_ptr(), losses.numel(), n_domains,
                                         sums.data_ptr(), counts.data_ptr(), C.c_void_p(_lib.stream_ptr(stream))))
    return sums, counts


def allreduce_domain_loss(sums, counts, group=None):
    """Sum per-domain (loss, count) vectors across data-parallel ranks
    (PAPER.md:756-760): one NCCL all-reduce of a packed f64 [2K] buffer
    (counts are exact in f64 below 2^53)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return sums, counts
    buf = torch.cat([sums, counts.to(torch.float64)])
    dist.all_reduce(buf, group=group)
    k = sums.numel()
    return buf[:k].contiguous(), buf[k:].round().to(torch.int64)


@dataclass
class _DomainTrack:
    history: list = field(default_factory=list)
    law: DomainLaw | None = None
    last_loss: float | None = None
    carried: int = 0


class AdoState:
    """Mutable ADO state of one job (``ado.py:179-376``); vectors live in HBM."""

    def __init__(self, config: AdoConfig, prior: Mapping[MixtureKey, float], device="cuda"):
        import torch

        total = sum(prior.values())
        if abs(total - 1.0) > 1e-9:
            raise MixtureError(f"prior must sum to 1, got {total!r}")
        self.config = config
        self.domains: list[MixtureKey] = sorted_keys(prior)
        if len(self.domains) < 2:
            raise MixtureError("adaptive optimization needs at least 2 domains")
        self.p_min = config.resolved_p_min(len(self.domains))
        self.device = torch.device(device)
        mu = np.array([float(prior[k]) for k in self.domains], dtype=np.float64)
        self._mu = torch.from_numpy(mu).to(self.device)
        self._credit = self._mu.clone()
        self._pi = self._mu.clone()
        self._pi_bar = self._mu.clone()
        self._pi_bar_count = torch.ones(1, dtype=torch.int64, device=self.device)
        self._law = torch.full((len(self.domains), 4), float("nan"), dtype=torch.float64, device=self.device)
        self.t = 0
        self.cumulative_samples = 0
        self._cum_at_step: list[int] = []
        self.tracks = {k: _DomainTrack() for k in self.domains}
        self.fit_steps: list[int] = []

    # -- dict views of the device vectors (reference attribute names)
    def _as_dict(self, t) -> dict:
        return dict(zip(self.domains, t.cpu().tolist()))

    @property
    def mu(self) -> dict:
        return self._as_dict(self._mu)

    @property
    def credit(self) -> dict:
        return self._as_dict(self._credit)

    @credit.setter
    def credit(self, d) -> None:
        self._set(self._credit, d)

    @property
    def pi(self) -> dict:
        return self._as_dict(self._pi)

    @pi.setter
    def pi(self, d) -> None:
        self._set(self._pi, d)

    @property
    def pi_bar(self) -> dict:
        return self._as_dict(self._pi_bar)

    @pi_bar.setter
    def pi_bar(self, d) -> None:
        self._set(self._pi_bar, d)

    @property
    def _pi_bar_count_value(self) -> int:
        return int(self._pi_bar_count.item())

    def _set(self, t, d) -> None:
        import torch

        t.copy_(torch.tensor([float(d[k]) for k in self.domains], dtype=torch.float64))

    @property
    def fitted(self) -> bool:
        return bool(self.fit_steps)

    # -------------------------------------------------------------- feedback
    def record_step(self, step: int, losses: Mapping[MixtureKey, float], num_samples: int | None = None) -> None:
        if step != self.t + 1:
            raise FeedbackError(f"expected step {self.t + 1}, got {step}")
        unknown = set(losses) - set(self.domains)
        if unknown:
            raise FeedbackError(f"unknown domain in losses: {sorted(unknown, key=MixtureKey.sort_key)[0]}")
        self.t = step
        self.cumulative_samples += self.config.samples_per_step if num_samples is None else int(num_samples)
        self._cum_at_step.append(self.cumulative_samples)
        for key in self.domains:
            tr = self.tracks[key]
            if key in losses:
                tr.last_loss = float(losses[key])
                tr.history.append((step, tr.last_loss))
            else:
                tr.carried += 1
                if tr.last_loss is not None:
                    tr.history.append((step, tr.last_loss))
        _lib.check(_lib.lib().mx_ado_credit(len(self.domains), float(self.config.credit_rate),
                                            self._pi.data_ptr(), self._credit.data_ptr(),
                                            C.c_void_p(_lib.stream_ptr())))
        cfg = self.config
        if step >= cfg.fit_start_step and step % cfg.refit_every == 0:
            self._refit(step)

    def _shared_n(self, step: int) -> float:
        if 1 <= step <= len(self._cum_at_step):
            total = self._cum_at_step[step - 1]
        else:
            total = self.cumulative_samples
        return max(total / len(self.domains), 1.0)

    def _refit(self, step: int) -> None:
        import torch

        cfg = self.config
        todo, hist = [], []
        for i, key in enumerate(self.domains):
            pts = [(self._shared_n(s), v) for s, v in self.tracks[key].history
                   if s > cfg.discard_first and s % cfg.subsample_every == 0]
            if len(pts) < 8:
                logger.warning("domain %s: only %d usable points, fit skipped", key, len(pts))
                continue
            todo.append(i)
            hist.append(pts)
        if todo:
            laws = fit_power_laws(hist, self.device)
            for i, law in zip(todo, laws):
                self.tracks[self.domains[i]].law = law
            rows = torch.tensor([[l.epsilon, l.beta, l.alpha, float(l.fallback)] for l in laws],
                                dtype=torch.float64, device=self.device)
            self._law[torch.tensor(todo, device=self.device)] = rows
        self.fit_steps.append(step)

    # -------------------------------------------------------------------- pi
    def compute_pi(self) -> dict[MixtureKey, float]:
        if not self.fitted:
            return self.mu
        L = _lib.lib()
        _lib.check(L.mx_ado_pi(len(self.domains), self._mu.data_ptr(), self._credit.data_ptr(),
                               self._law.data_ptr(), float(self._shared_n(self.t)), float(self.p_min),
                               float(self.config.smoothing), self._pi_bar.data_ptr(),
                               self._pi_bar_count.data_ptr(), self._pi.data_ptr(),
                               C.c_void_p(_lib.stream_ptr())))
        return self.pi

    def _floored(self, dist: Mapping[MixtureKey, float]) -> dict[MixtureKey, float]:
        """_floored (ado.py:273-291) via the device kernel: a fitted-free state
        with zero credit reduces compute_pi to floor(mu)."""
        import torch

        k = len(self.domains)
        mu = torch.tensor([float(dist[x]) for x in self.domains], dtype=torch.float64, device=self.device)
        zero = torch.zeros(k, dtype=torch.float64, device=self.device)
        law = torch.full((k, 4), float("nan"), dtype=torch.float64, device=self.device)
        out = torch.empty(k, dtype=torch.float64, device=self.device)
        cnt = torch.ones(1, dtype=torch.int64, device=self.device)
        _lib.check(_lib.lib().mx_ado_pi(k, mu.data_ptr(), zero.data_ptr(), law.data_ptr(), 1.0,
                                        float(self.p_min), 0.0, zero.clone().data_ptr(), cnt.data_ptr(),
                                        out.data_ptr(), C.c_void_p(_lib.stream_ptr())))
        return dict(zip(self.domains, out.cpu().tolist()))

    # ------------------------------------------------------------ checkpoint
    def state_dict(self) -> dict:
        def dist(d):
            return {k.canonical_string(): d[k] for k in self.domains}

        return {
            "config": self.config.to_json(),
            "mu": dist(self.mu),
            "t": self.t,
            "cumulative_samples": self.cumulative_samples,
            "cum_at_step": list(self._cum_at_step),
            "credit": dist(self.credit),
            "pi": dist(self.pi),
            "pi_bar": dist(self.pi_bar),
            "pi_bar_count": self._pi_bar_count_value,
            "fit_steps": list(self.fit_steps),
            "tracks": {
                k.canonical_string(): {
                    "history": self.tracks[k].history,
                    "law": None if self.tracks[k].law is None else {
                        "epsilon": self.tracks[k].law.epsilon, "beta": self.tracks[k].law.beta,
                        "alpha": self.tracks[k].law.alpha, "fallback": self.tracks[k].law.fallback},
                    "last_loss": self.tracks[k].last_loss,
                    "carried": self.tracks[k].carried,
                }
                for k in self.domains
            },
        }

    @staticmethod
    def from_state(state: Mapping, device="cuda") -> "AdoState":
        import torch

        config = AdoConfig.from_json(state["config"])
        mu = {MixtureKey.parse(k): v for k, v in state["mu"].items()}
        out = AdoState(config, mu, device)
        out.t = int(state["t"])
        out.cumulative_samples = int(state["cumulative_samples"])
        out._cum_at_step = [int(v) for v in state.get("cum_at_step", [])]
        out.credit = {MixtureKey.parse(k): float(v) for k, v in state["credit"].items()}
        out.pi = {MixtureKey.parse(k): float(v) for k, v in state["pi"].items()}
        out.pi_bar = {MixtureKey.parse(k): float(v) for k, v in state["pi_bar"].items()}
        out._pi_bar_count.fill_(int(state["pi_bar_count"]))
        out.fit_steps = [int(s) for s in state["fit_steps"]]
        for ks, tr in state["tracks"].items():
            key = MixtureKey.parse(ks)
            track = out.tracks[key]
            track.history = [(int(s), float(l)) for s, l in tr["history"]]
            law = tr["law"]
            track.law = None if law is None else DomainLaw(**law)
            track.last_loss = tr["last_loss"]
            track.carried = int(tr["carried"])
            if track.law is not None:
                i = out.domains.index(key)
                out._law[i] = torch.tensor([track.law.epsilon, track.law.beta, track.law.alpha,
                                            float(track.law.fallback)], dtype=torch.float64)
        return out


class AdoSource(MixtureSource):
    """Mixture provider backed by a device AdoState (``ado.py:379-409``)."""

    algorithm = "ado"

    def __init__(self, state: AdoState, chunk_size: int):
        self.state = state
        self.chunk_size = int(chunk_size)

    def current_spec(self) -> MixtureSpec:
        return MixtureSpec(self.state.compute_pi(), self.chunk_size)

    def observe_feedback(self, step: int, losses: Mapping[MixtureKey, tuple[float, int]]) -> None:
        means = {k: float(t) / int(c) for k, (t, c) in losses.items() if int(c) > 0}
        counts = sum(int(v[1]) for v in losses.values())
        self.state.record_step(step, means, num_samples=counts or None)

    def is_dynamic(self) -> bool:
        return True

    def state_dict(self) -> dict:
        return {"ado": self.state.state_dict(), "chunk_size": self.chunk_size}

    def load_state(self, state: Mapping) -> None:
        self.state = AdoState.from_state(state["ado"])
        self.chunk_size = int(state["chunk_size"])
