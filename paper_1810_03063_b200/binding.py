"""Thin ctypes binding of the C ABI in include/egt_b200.h (argument marshalling only).

Every computation happens in the CUDA library ``lib/libegt_b200.so``; if it is
missing or cannot find a CUDA device, calls raise ``EGTError`` -- there is no
CPU fallback.  Device buffers are passed as anything with ``data_ptr()``
(torch CUDA tensors) or as raw integer addresses.
"""
import ctypes
import os
from fractions import Fraction

import numpy as np

from . import build as _build

KUHN, LEDUC, RIVER = 1, 2, 3
EGT_THEORY, EGT_BALANCED, EGT_AS = 0, 1, 2
CFR_RM, CFR_RMP, CFR_PLUS = 0, 1, 2
CONTEXTS = ("P1_OPEN", "P1_VS_BET", "P1_VS_RAISE", "P1_SUBSEQ",
            "P2_VS_CHECK", "P2_VS_BET", "P2_SUBSEQ")
N_CTX, MAX_FRACS = 7, 16


class EGTError(RuntimeError):
    pass


class Spec(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("n_games", ctypes.c_int32),
        ("pot", ctypes.c_int32), ("stack", ctypes.c_int32),
        ("raise_cap", ctypes.c_int32), ("open_fold", ctypes.c_int32),
        ("n_fracs", ctypes.c_int32 * N_CTX),
        ("frac_num", (ctypes.c_int32 * MAX_FRACS) * N_CTX),
        ("frac_den", (ctypes.c_int32 * MAX_FRACS) * N_CTX),
        ("allin", ctypes.c_int32 * N_CTX),
        ("n_ranks", ctypes.c_int32), ("n_suits", ctypes.c_int32),
        ("boards", ctypes.POINTER(ctypes.c_int32)),
        ("prior1", ctypes.POINTER(ctypes.c_double)),
        ("prior2", ctypes.POINTER(ctypes.c_double)),
        ("precision", ctypes.c_int32),
    ]


class Info(ctypes.Structure):
    _fields_ = [
        ("n_games", ctypes.c_int32), ("H", ctypes.c_int32), ("H_pad", ctypes.c_int32),
        ("n_combos", ctypes.c_int32), ("n_pub", ctypes.c_int32 * 2), ("n_nodes", ctypes.c_int32 * 2),
        ("n_terminals", ctypes.c_int32), ("depth", ctypes.c_int32 * 2),
        ("vec_stride", ctypes.c_int64 * 2), ("max_abs_A", ctypes.c_double * 1),
        ("h2d_bytes", ctypes.c_int64),
        ("grad_rows_read", ctypes.c_int32 * 2), ("grad_rows_written", ctypes.c_int32 * 2),
        ("precision", ctypes.c_int32),
    ]


EXPORTS = [
    "egt_load_game", "egt_free_game", "egt_set_stream", "egt_game_info_get", "egt_hand_cards",
    "egt_pub_history", "egt_gradient", "egt_smoothed_br", "egt_prox", "egt_best_response",
    "egt_init", "egt_step", "cfr_init", "cfr_step", "saddle_gap", "get_avg_strategy",
    "get_strategy_device", "egt_scalars", "egt_last_error", "saddle_gap_device",
    "egt_timing", "egt_timing_get", "egt_nccl_unique_id", "egt_shard", "egt_gradient_rows",
    "egt_ipc_handles", "egt_shard_peers", "egt_gradient_rows_to", "egt_pool_trim", "egt_set_target",
    "egt_shard_emulate",
]
IPC_HANDLE_BYTES = 64
KERNEL_KINDS = ("grad_Ay", "grad_ATx", "tree", "scalar", "comm")
NCCL_ID_BYTES = 128

_lib = None


def lib_path():
    return _build.LIB


def load_library():
    """Load the CUDA library (fails loudly if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        raise EGTError("CUDA library not built: %s (run python -m paper_1810_03063_b200.build)" % path)
    L = ctypes.CDLL(path)
    P, I32, I64, D, VP = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p
    sig = {
        "egt_load_game": ([ctypes.POINTER(Spec), ctypes.POINTER(P)], I32),
        "egt_free_game": ([P], None),
        "egt_set_stream": ([P, VP], I32),
        "egt_game_info_get": ([P, ctypes.POINTER(Info)], I32),
        "egt_hand_cards": ([P, I32, ctypes.POINTER(I32)], I32),
        "egt_pub_history": ([P, I32, I32, ctypes.c_char_p, I32], I32),
        "egt_gradient": ([P, I32, VP, VP], I32),
        "egt_smoothed_br": ([P, I32, VP, D, VP, VP, VP, VP, VP], I32),
        "egt_prox": ([P, I32, VP, D, VP, VP, VP], I32),
        "egt_best_response": ([P, I32, VP, D, VP], I32),
        "egt_init": ([P, I32, D, D], I32),
        "egt_step": ([P, I32], I32),
        "cfr_init": ([P, I32], I32),
        "cfr_step": ([P, I32], I32),
        "saddle_gap": ([P, I32, ctypes.POINTER(D)], I32),
        "get_avg_strategy": ([P, I32, ctypes.POINTER(D)], I32),
        "get_strategy_device": ([P, I32, I32, VP], I32),
        "egt_scalars": ([P, ctypes.POINTER(D)], I32),
        "egt_last_error": ([], ctypes.c_char_p),
        "egt_pool_trim": ([], I32),
        "egt_set_target": ([P, ctypes.POINTER(D)], I32),
        "saddle_gap_device": ([P, I32, VP], I32),
        "egt_timing": ([P, I32], I32),
        "egt_timing_get": ([P, ctypes.POINTER(D)], I32),
        "egt_nccl_unique_id": ([ctypes.c_char_p], I32),
        "egt_shard": ([P, I32, I32, ctypes.c_char_p], I32),
        "egt_gradient_rows": ([P, I32, I32, I32, VP, VP], I32),
        "egt_ipc_handles": ([P, ctypes.c_char_p], I32),
        "egt_shard_peers": ([P, ctypes.c_char_p], I32),
        "egt_gradient_rows_to": ([P, I32, I32, I32, VP, ctypes.POINTER(ctypes.c_uint64), I32], I32),
        "egt_shard_emulate": ([P, I32, I32], I32),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    del I64
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        raise EGTError("egt_b200 error %d: %s" % (rc, _lib.egt_last_error().decode()))


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


F64, F32 = 0, 1


def _spec_from(kind, n_games, river, boards, prior1, prior2, n_ranks, n_suits, precision=F64):
    s = Spec()
    s.kind = kind
    s.n_games = n_games
    s.precision = {"f64": F64, "f32": F32}.get(precision, precision)
    keep = []
    if kind == RIVER:
        s.pot, s.stack = river["pot"], river["stack"]
        s.raise_cap = river["raise_cap"] if river["raise_cap"] < 10 ** 6 else 0
        s.open_fold = int(river["open_fold"])
        for c, ctx in enumerate(CONTEXTS):
            fr = [Fraction(f) for f in river["fracs"].get(ctx, ())]
            s.n_fracs[c] = len(fr)
            for i, f in enumerate(fr):
                s.frac_num[c][i], s.frac_den[c][i] = f.numerator, f.denominator
            s.allin[c] = int(river["allin"].get(ctx, False))
        s.n_ranks, s.n_suits = n_ranks, n_suits
        b = np.ascontiguousarray(boards, dtype=np.int32).reshape(n_games, 5)
        keep.append(b)
        s.boards = b.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        for name, pr in (("prior1", prior1), ("prior2", prior2)):
            if pr is not None:
                a = np.ascontiguousarray(pr, dtype=np.float64)
                keep.append(a)
                setattr(s, name, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return s, keep


class Game:
    """A batch of games sharing one public tree (C ABI handle ``egt_game``)."""

    def __init__(self, kind, n_games=1, river=None, boards=None, prior1=None, prior2=None,
                 n_ranks=13, n_suits=4, precision="f64"):
        """precision: "f64" (default) or "f32" (the optional fp32 mode): element type of every
        device vector of this game."""
        L = load_library()
        spec, keep = _spec_from(kind, n_games, river, boards, prior1, prior2, n_ranks, n_suits, precision)
        h = ctypes.c_void_p()
        _check(L.egt_load_game(ctypes.byref(spec), ctypes.byref(h)))
        del keep
        self._h = h
        self._L = L
        info = Info()
        _check(L.egt_game_info_get(h, ctypes.byref(info)))
        self.n_games = info.n_games
        self.H, self.H_pad, self.n_combos = info.H, info.H_pad, info.n_combos
        self.n_pub = (info.n_pub[0], info.n_pub[1])
        self.n_nodes = (info.n_nodes[0], info.n_nodes[1])
        self.depth = (info.depth[0], info.depth[1])
        self.n_terminals = info.n_terminals
        self.vec_stride = (info.vec_stride[0], info.vec_stride[1])
        self.h2d_bytes = info.h2d_bytes
        self.grad_rows_read = (info.grad_rows_read[0], info.grad_rows_read[1])
        self.grad_rows_written = (info.grad_rows_written[0], info.grad_rows_written[1])
        self.precision = "f32" if info.precision == F32 else "f64"
        self.np_dtype = np.float32 if self.precision == "f32" else np.float64

    def close(self):
        if self._h:
            self._L.egt_free_game(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- layout
    def set_stream(self, stream):
        """cudaStream_t (int), a torch.cuda.Stream, or None (legacy default stream)."""
        if stream is not None and not isinstance(stream, int):
            stream = stream.cuda_stream
        _check(self._L.egt_set_stream(self._h, stream))

    def hand_cards(self, g):
        out = (ctypes.c_int32 * (2 * self.H))()
        _check(self._L.egt_hand_cards(self._h, g, out))
        return np.frombuffer(out, dtype=np.int32).reshape(self.H, 2).copy()

    def pub_history(self, player, s):
        buf = ctypes.create_string_buffer(4096)
        _check(self._L.egt_pub_history(self._h, player, s, buf, 4096))
        return buf.value.decode()

    def vec_shape(self, player):
        return (self.n_games, self.n_pub[player], self.H_pad)

    @property
    def torch_dtype(self):
        import torch
        return torch.float32 if self.precision == "f32" else torch.float64

    # ---- kernel-level calls (device buffers)
    def egt_gradient(self, player, din, dout):
        _check(self._L.egt_gradient(self._h, player, _ptr(din), _ptr(dout)))

    def egt_smoothed_br(self, player, g, gsign, mu, q=None, b=None, value=None, lb=None):
        _check(self._L.egt_smoothed_br(self._h, player, _ptr(g), float(gsign), _ptr(mu),
                                       _ptr(q), _ptr(b), _ptr(lb), _ptr(value)))

    def egt_prox(self, player, g, gsign, step, center_lb, q):
        """center_lb: the centre's behavioural strategy as natural logs (R16)."""
        _check(self._L.egt_prox(self._h, player, _ptr(g), float(gsign), _ptr(step), _ptr(center_lb), _ptr(q)))

    def egt_best_response(self, player, g, gsign, value):
        _check(self._L.egt_best_response(self._h, player, _ptr(g), float(gsign), _ptr(value)))

    # ---- solvers
    def egt_init(self, variant, mu_x=0.0, mu_y=0.0):
        _check(self._L.egt_init(self._h, variant, float(mu_x), float(mu_y)))

    def egt_set_target(self, eps):
        """Per-game eps_sad target (scalar or [n_games], payoff units; None clears) at which
        an EGT/as game stops iterating, decided on the device (egt_set_target)."""
        if eps is None:
            _check(self._L.egt_set_target(self._h, None))
            return
        t = np.ascontiguousarray(np.broadcast_to(np.asarray(eps, dtype=np.float64), (self.n_games,)))
        _check(self._L.egt_set_target(self._h, t.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))

    def egt_step(self, n=1):
        _check(self._L.egt_step(self._h, n))

    def cfr_init(self, variant):
        _check(self._L.cfr_init(self._h, variant))

    def cfr_step(self, n=1):
        _check(self._L.cfr_step(self._h, n))

    def saddle_gap(self, which=0, out=None):
        """Host fp64 [n_games]; `out` may be a preallocated (pinned) float64 buffer."""
        if out is None:
            out = np.zeros(self.n_games)
        _check(self._L.saddle_gap(self._h, which, ctypes.cast(_host_ptr(out), ctypes.POINTER(ctypes.c_double))))
        return out

    def saddle_gap_device(self, which, dout):
        """Per-game eps_sad into a DEVICE fp64 [n_games] buffer, stream-ordered."""
        _check(self._L.saddle_gap_device(self._h, which, _ptr(dout)))

    def gradient_rows(self, player, rank, world, din, dout):
        """Rows shard `rank` of `world` computes (others 0), no communication."""
        _check(self._L.egt_gradient_rows(self._h, player, rank, world, _ptr(din), _ptr(dout)))

    def shard(self, rank, world, uid=None):
        """Shard every gradient of this game over `world` ranks (C ABI egt_shard).  `uid`: the
        NCCL unique id bytes from rank 0 (``nccl_unique_id``); with torch.distributed
        initialised and uid None, rank 0 makes it and broadcasts it (host-side plumbing)."""
        if world > 1 and uid is None:
            uid = broadcast_uid(nccl_unique_id() if rank == 0 else None)
        buf = None if uid is None else ctypes.create_string_buffer(bytes(uid), NCCL_ID_BYTES)
        _check(self._L.egt_shard(self._h, rank, world, buf))

    def shard_emulate(self, world, fused=False):
        """Emulate `world` ranks on this device (egt_shard_emulate; tests)."""
        _check(self._L.egt_shard_emulate(self._h, world, int(bool(fused))))

    def gradient_rows_to(self, player, rank, world, din, dsts):
        """Shard `rank`'s rows stored into every buffer of dsts (the fused all-gather's stores)."""
        arr = (ctypes.c_uint64 * len(dsts))(*[_ptr(d) for d in dsts])
        _check(self._L.egt_gradient_rows_to(self._h, player, rank, world, _ptr(din), arr, len(dsts)))

    def ipc_handles(self):
        buf = ctypes.create_string_buffer(2 * IPC_HANDLE_BYTES)
        _check(self._L.egt_ipc_handles(self._h, buf))
        return buf.raw

    def shard_peers(self, all_handles):
        """all_handles: bytes of every rank's ipc_handles() in rank order (fused all-gather)."""
        blob = b"".join(all_handles)
        _check(self._L.egt_shard_peers(self._h, ctypes.create_string_buffer(blob, len(blob))))

    def shard_fused(self, rank, world):
        """egt_shard + egt_shard_peers over an initialised torch.distributed group: rank 0's
        NCCL id and every rank's IPC handles travel over the host-side group."""
        import torch.distributed as dist
        self.shard(rank, world)
        handles = [None] * world
        dist.all_gather_object(handles, self.ipc_handles())
        self.shard_peers(handles)

    def timing(self, enable):
        _check(self._L.egt_timing(self._h, int(bool(enable))))

    def timing_get(self):
        """{kind: (ms, launches, active game-launches, algorithmic bytes)} since timing(True)."""
        out = np.zeros(4 * len(KERNEL_KINDS))
        _check(self._L.egt_timing_get(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return {k: tuple(out[4 * i:4 * i + 4]) for i, k in enumerate(KERNEL_KINDS)}

    def get_avg_strategy(self, player, out=None):
        if out is None:
            out = np.zeros((self.n_games, self.n_pub[player], self.n_combos))
        _check(self._L.get_avg_strategy(self._h, player,
                                        ctypes.cast(_host_ptr(out), ctypes.POINTER(ctypes.c_double))))
        return out

    def get_strategy_device(self, player, which, dout):
        _check(self._L.get_strategy_device(self._h, player, which, _ptr(dout)))

    def egt_scalars(self):
        out = np.zeros((self.n_games, 8))
        _check(self._L.egt_scalars(self._h, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return out


def _host_ptr(a):
    if isinstance(a, np.ndarray):
        assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    return a.data_ptr()  # pinned torch CPU tensor


def pool_trim():
    """Give the memory the library's device pool keeps from freed games back to the driver
    (egt_pool_trim); live games keep theirs."""
    _check(load_library().egt_pool_trim())


def nccl_unique_id():
    """C ABI egt_nccl_unique_id: NCCL_ID_BYTES bytes (rank 0 makes it, all ranks use it)."""
    L = load_library()
    buf = ctypes.create_string_buffer(NCCL_ID_BYTES)
    _check(L.egt_nccl_unique_id(buf))
    return buf.raw


def broadcast_uid(uid):
    """Rank 0's NCCL unique id to every rank over the initialised torch.distributed group."""
    import torch.distributed as dist
    box = [uid]
    dist.broadcast_object_list(box, src=0)
    assert box[0] is not None and len(box[0]) == NCCL_ID_BYTES
    return box[0]


def load_game(kind, **kw):
    """C ABI ``egt_load_game``."""
    return Game(kind, **kw)
