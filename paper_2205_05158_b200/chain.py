"""Device-resident state and one step of the hot path, on top of the C ABI.

``Chain`` owns the per-run device tensors (CNN params, PA coefficients, channel,
ZF precoder, workspaces) and runs one step over a batch of OFDM symbols:

    fdcnn_forward (a1) -> chain_tx (a3+a4+a5 fused) -> ue_receive_ser (a6)

with the ZF build (a2) done once per channel realisation at construction
(SURVEY.md §8(c) reading A10).  Pure orchestration: every arithmetic step is a
libfdpd.so kernel.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import fdpd


@dataclass
class Shapes:
    U: int
    B: int
    N_d: int
    N_ifft: int
    M_qam: int
    chans: tuple
    orders: tuple
    L: int
    M: int
    rho: float = 0.3
    eps: float = 1e-4
    head: str = "residual"      # FD-CNN variant: BASELINE residual stack or the paper's conv + FC head
    n_conv: int = 2

    @classmethod
    def from_config(cls, cfg):
        return cls(U=cfg.U, B=cfg.B, N_d=cfg.N_d, N_ifft=cfg.N_ifft, M_qam=cfg.M_qam, chans=tuple(cfg.chans),
                   orders=tuple(cfg.orders), L=cfg.L, M=cfg.M, rho=cfg.rho, head=cfg.head, n_conv=cfg.n_conv)


class Chain:
    def __init__(self, shapes: Shapes, h_taps, coef, params, device="cuda", max_batch=1, b0=0, B_loc=None,
                 impair=None, precode_math="auto"):
        """impair (NEXT f3, optional): dict with clip, pa_noise_std, awgn_n0, csi_eta, noise_key, h_err.
        precode_math (split path): "simt" FP32 SIMT, "tf32" TF32 tensor cores, "fp32tc" FP32-accurate
        split-TF32 tensor cores (the latter two on the precode_pack'ed precoder); "auto" = fdpd.auto_precode_math
        (fp32tc where the tensor-core kernel applies: the split path with U % 4 == 0, U <= 32)."""
        self.sh = shapes
        self.device = torch.device(device)
        dev = self.device
        self.b0 = b0
        self.B_loc = shapes.B - b0 if B_loc is None else B_loc
        self.h_taps = torch.as_tensor(h_taps).to(dev, torch.complex64).contiguous()
        self.coef = torch.as_tensor(coef).to(dev, torch.complex64)[b0:b0 + self.B_loc].contiguous()
        self.params = torch.as_tensor(params).to(dev, torch.float32).contiguous()
        self.impair = dict(impair) if impair else None
        # precode as its own tiled kernel (then chain_txrx_pre) from U >= 16: the fused prologue
        # gathers U P_b and s_n rows per (symbol, antenna) CTA from L2, which dominates at
        # C4/C5 (measured: C4 17.7 -> 13.8 ms, C5 11.5 -> 7.4 ms) but not at C2/C3 (U <= 8)
        self.split_precode = shapes.U >= fdpd.SPLIT_PRECODE_MIN_U
        # a2, once per channel realisation
        if self.impair and self.impair.get("csi_eta", 0.0) > 0:
            h_err = torch.as_tensor(self.impair["h_err"]).to(dev, torch.complex64).contiguous()
            self.h_fd, self.P, self.alpha = fdpd.zf_precoder_build_ex(self.h_taps, h_err, self.impair["csi_eta"],
                                                                      shapes.N_ifft, shapes.N_d, shapes.rho, b0=b0,
                                                                      B_loc=self.B_loc)
        else:
            self.h_fd, self.P, self.alpha = fdpd.zf_precoder_build(self.h_taps, shapes.N_ifft, shapes.N_d,
                                                                   shapes.rho, b0=b0, B_loc=self.B_loc)
        self.precode_math = fdpd.auto_precode_math(shapes.U) if precode_math == "auto" else precode_math
        self.Ppk = fdpd.precode_pack(self.P) if self.precode_math != "simt" else None
        self.reserve(max_batch)

    def _imp(self, sym0):
        i = self.impair or {}
        return fdpd.make_impairments(i.get("clip", 0.0), i.get("pa_noise_std", 0.0), i.get("awgn_n0", 0.0),
                                     i.get("csi_eta", 0.0), i.get("noise_key", 0), sym0, self.b0, self.sh.B)

    def reserve(self, n):
        sh, dev = self.sh, self.device
        self.cap = n
        self.s_tilde = torch.empty((n, sh.U, sh.N_d), dtype=torch.complex64, device=dev)
        self.y = torch.empty((n, self.B_loc, sh.N_ifft), dtype=torch.complex64, device=dev)
        self.yhat = torch.empty((n, sh.U, sh.N_d), dtype=torch.complex64, device=dev)
        self.counts = torch.zeros(3, dtype=torch.int64, device=dev)
        if sh.head == "paper":
            need = fdpd.lib().fdcnn_paper_workspace_bytes(sh.n_conv, n, sh.U, sh.N_d)
        else:
            need = fdpd.lib().fdcnn_workspace_bytes(fdpd._ints(sh.chans), len(sh.chans) - 1, n, sh.U, sh.N_d)
        self.ws_cnn = fdpd._ws(need, self.y)
        self.ws_rx = fdpd._ws(fdpd.lib().ue_receive_workspace_bytes(n, self.B_loc, sh.N_d), self.y)

    # ------------------------------------------------------------------ stages
    def dpd(self, s):
        n = s.shape[0]
        if self.sh.head == "paper":
            return fdpd.fdcnn_paper_forward(self.params, self.sh.n_conv, s, out=self.s_tilde[:n],
                                            workspace=self.ws_cnn)
        return fdpd.fdcnn_forward(self.params, self.sh.chans, s, out=self.s_tilde[:n], workspace=self.ws_cnn)

    def tx(self, s_tilde):
        n = s_tilde.shape[0]
        sh = self.sh
        return fdpd.chain_tx(self.P, s_tilde, self.coef, sh.orders, sh.L, sh.M, sh.N_ifft, out=self.y[:n])

    def rx(self, y, tx_idx, counts=None, dec=None):
        """Unfused evaluation from the stored waveform: receive FFT + channel sum + SER."""
        n = y.shape[0]
        sh = self.sh
        counts = self.counts if counts is None else counts
        return fdpd.ue_receive_ser(y, self.h_fd, self.alpha, tx_idx, sh.M_qam, yhat=self.yhat[:n], counts=counts,
                                   dec=dec, workspace=self.ws_rx, boundary_eps=sh.eps)

    def txrx(self, s_tilde, sym0=0):
        """Fused precode -> IDFT -> GMP (waveform stored) -> receive DFT at the data bins."""
        n = s_tilde.shape[0]
        sh = self.sh
        XPA = self.ws_rx[: 8 * n * self.B_loc * sh.N_d].view(torch.complex64).view(n, self.B_loc, sh.N_d)
        if self.split_precode:
            # precode as its own kernel, then the fused chain on X
            return self.txrx_pre(self.precode(s_tilde), sym0)
        if self.impair:
            return fdpd.chain_txrx_ex(self.P, s_tilde, self.coef, sh.orders, sh.L, sh.M, sh.N_ifft, self._imp(sym0),
                                      y=self.y[:n], XPA=XPA)
        return fdpd.chain_txrx(self.P, s_tilde, self.coef, sh.orders, sh.L, sh.M, sh.N_ifft, y=self.y[:n], XPA=XPA)

    def precode(self, s_tilde):
        """a3 on its own (the split path): X = precode(P, s_tilde) into the plan's buffer."""
        n = s_tilde.shape[0]
        if getattr(self, "X", None) is None or self.X.shape[0] < n:
            self.X = torch.empty((max(n, self.cap), self.B_loc, self.sh.N_d), dtype=torch.complex64,
                                 device=self.device)
        if self.Ppk is not None:
            return fdpd.precode_packed(self.Ppk, s_tilde, out=self.X[:n], math=fdpd.MATH[self.precode_math])
        return fdpd.precode(self.P, s_tilde, out=self.X[:n])

    def txrx_pre(self, X, sym0=0):
        """IDFT -> GMP (waveform stored) -> receive DFT on a precoded spectrum X (split path)."""
        n = X.shape[0]
        sh = self.sh
        XPA = self.ws_rx[: 8 * n * self.B_loc * sh.N_d].view(torch.complex64).view(n, self.B_loc, sh.N_d)
        return fdpd.chain_txrx_pre(X, self.coef, sh.orders, sh.L, sh.M, sh.N_ifft,
                                   imp=self._imp(sym0) if self.impair else None, y=self.y[:n], XPA=XPA)

    def combine(self, XPA, tx_idx, counts=None, dec=None, sym0=0):
        n = XPA.shape[0]
        sh = self.sh
        counts = self.counts if counts is None else counts
        if self.impair:
            return fdpd.ue_combine_ser_ex(XPA, self.h_fd, self.alpha, tx_idx, sh.M_qam, self._imp(sym0),
                                          yhat=self.yhat[:n], counts=counts, dec=dec, boundary_eps=sh.eps)
        return fdpd.ue_combine_ser(XPA, self.h_fd, self.alpha, tx_idx, sh.M_qam, yhat=self.yhat[:n], counts=counts,
                                   dec=dec, boundary_eps=sh.eps)

    def step_redraw(self, s, tx_idx, h_taps_all, counts=None, dec=None, sym0=0):
        """One step with per-symbol channel redraw (NEXT f4): the batched ZF build joins the
        hot path.  h_taps_all [n][T][U][B] on the device.
        fdcnn_forward -> zf_precoder_build_batched -> chain_txrx_ps -> ue_combine_ser_ps."""
        if s.shape[0] > self.cap:
            self.reserve(s.shape[0])
        st = self.dpd(s)
        XPA = self.redraw_txrx(st, h_taps_all, sym0)
        return self.redraw_combine(XPA, tx_idx, counts=counts, dec=dec, sym0=sym0)

    def redraw_txrx(self, s_tilde, h_taps_all, sym0=0):
        """Batched per-symbol ZF build, then chain_txrx_ps."""
        n = s_tilde.shape[0]
        sh = self.sh
        if getattr(self, "_zfb_n", None) != n:
            self._zfb = None
            self._zfb_n = n
        self._zfb = fdpd.zf_precoder_build_batched(h_taps_all, sh.N_ifft, sh.N_d, sh.rho, out=self._zfb)
        self.h_fd_all, self.P_all, self.alpha_all, self.zf_status, _ = self._zfb
        imp = self._imp(sym0) if self.impair else None
        XPA = self.ws_rx[: 8 * n * self.B_loc * sh.N_d].view(torch.complex64).view(n, self.B_loc, sh.N_d)
        fdpd.chain_txrx_ps(self.P_all, s_tilde, self.coef, sh.orders, sh.L, sh.M, sh.N_ifft, imp=imp,
                           y=self.y[:n], XPA=XPA)
        return XPA

    def redraw_combine(self, XPA, tx_idx, counts=None, dec=None, sym0=0):
        n = XPA.shape[0]
        sh = self.sh
        imp = self._imp(sym0) if self.impair else None
        counts = self.counts if counts is None else counts
        return fdpd.ue_combine_ser_ps(XPA, self.h_fd_all, self.alpha_all, tx_idx, sh.M_qam, imp=imp,
                                      yhat=self.yhat[:n], counts=counts, dec=dec, boundary_eps=sh.eps)

    def step(self, s, tx_idx, counts=None, dec=None, fused=True, sym0=0):
        """One pass of the hot path over a batch (s, tx_idx on the device; sym0 = global index of
        the batch's first symbol, used by the impairment noise):
        fdcnn_forward -> chain_txrx -> ue_combine_ser   (fused=True, 3 libfdpd calls)
        fdcnn_forward -> chain_tx -> ue_receive_ser     (fused=False, unimpaired only)."""
        if s.shape[0] > self.cap:
            self.reserve(s.shape[0])
        st = self.dpd(s)
        if not fused:
            if self.impair:
                raise ValueError("the unfused path has no impairment stages; use fused=True")
            return self.rx(self.tx(st), tx_idx, counts=counts, dec=dec)
        _, XPA = self.txrx(st, sym0)
        return self.combine(XPA, tx_idx, counts=counts, dec=dec, sym0=sym0)


class AntennaOps:
    """Per-rank compute of the Mode A step (dist.AntennaShardedStep) on the CUDA path: a Chain
    built on this rank's antenna rows [b0, b0 + B_loc) (zf_precoder_build emits only those rows
    from the replicated taps; alpha is the global one)."""

    def __init__(self, chain: Chain, events=None):
        self.ch = chain
        self.events = events          # optional list: (start, end) CUDA events around each chain launch

    def dpd(self, s, out):
        ch = self.ch
        if ch.sh.head == "paper":
            return fdpd.fdcnn_paper_forward(ch.params, ch.sh.n_conv, s, out=out, workspace=ch.ws_cnn)
        return fdpd.fdcnn_forward(ch.params, ch.sh.chans, s, out=out, workspace=ch.ws_cnn)

    def tx(self, st_all, XPA=None):
        """precode (split path) -> IDFT -> GMP (waveform into the plan's y) -> receive DFT."""
        ch, sh = self.ch, self.ch.sh
        n = st_all.shape[0]
        if XPA is None:
            XPA = torch.empty((n, ch.B_loc, sh.N_d), dtype=torch.complex64, device=ch.device)
        X = ch.precode(st_all)
        if self.events is not None:
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            ev[0].record()
        fdpd.chain_txrx_pre(X, ch.coef, sh.orders, sh.L, sh.M, sh.N_ifft, y=ch.y[:n], XPA=XPA)
        if self.events is not None:
            ev[1].record()
            self.events.append(ev)
        return XPA

    def combine(self, XPA, out):
        return fdpd.ue_combine(XPA, self.ch.h_fd, out=out)

    def slice(self, yhat, idx, counts):
        return fdpd.ue_slice_ser(yhat, self.ch.alpha, idx, self.ch.sh.M_qam, counts=counts,
                                 boundary_eps=self.ch.sh.eps)

    # fused exchange (dist.PeerExchange): partial sums stored into the owners' receive buffers
    def peer_ok(self):
        return 9 <= self.ch.sh.U <= 32 and self.ch.sh.N_d % 2 == 0

    def combine_peer(self, XPA, peer_recv, rank):
        return fdpd.ue_combine_peer(XPA, self.ch.h_fd, peer_recv, rank)

    def reduce_slice(self, recv, yhat, idx, counts):
        return fdpd.ue_reduce_ser(recv, self.ch.alpha, idx, self.ch.sh.M_qam, yhat=yhat, counts=counts,
                                  boundary_eps=self.ch.sh.eps)
