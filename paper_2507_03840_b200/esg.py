"""ctypes binding of libesg_b200.so (include/esg.h).

This mirrors the reference's C++ API names and argument meaning
(structures::build_graph, partition::lownn_partition, runtime::build_comm_plan,
model::Network<float>) so tests and the bench read like the reference's own
tests.  It is plumbing only: every computation runs inside the CUDA library,
and importing this module fails loudly if the library was not built.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libesg_b200.so")

OK, ERR_OTHER, ERR_USAGE, ERR_DATA, ERR_DIVERGENCE, ERR_NCCL, ERR_CUDA, ERR_OOM = range(8)
LINEAR_FP32, LINEAR_BF16 = 0, 1


class EsgError(RuntimeError):
    """Base of the mirrored esgnn::Error taxonomy (core/error.h:11-51)."""

    code = ERR_OTHER


class UsageError(EsgError):
    code = ERR_USAGE


class DataError(EsgError):
    code = ERR_DATA


class DivergenceError(EsgError):
    code = ERR_DIVERGENCE


class TransportError(EsgError):
    code = ERR_NCCL


class CudaError(EsgError):
    code = ERR_CUDA


class OutOfMemory(EsgError):
    code = ERR_OOM


_ERRORS = {c.code: c for c in (UsageError, DataError, DivergenceError, TransportError, CudaError, OutOfMemory)}

_lib_handle = None


class _Timing(C.Structure):
    _fields_ = [
        ("forward_ms", C.c_double),
        ("message_ms", C.c_double),
        ("halo_ms", C.c_double),
        ("heads_ms", C.c_double),
        ("exchanges", C.c_int64),
        ("gpu_launches", C.c_int64),
        ("halo_skew_ms", C.c_double),
        ("halo_exchange_ms", C.c_double),
        ("halo_bytes", C.c_int64),
    ]


class _ModelConfig(C.Structure):
    _fields_ = [
        ("l_max", C.c_int),
        ("e_width", C.c_int),
        ("layers", C.c_int),
        ("n_radial", C.c_int),
        ("r_cut", C.c_double),
        ("seed", C.c_uint64),
        ("gate_enabled", C.c_int),
        ("linear_precision", C.c_int),
    ]


def lib() -> C.CDLL:
    """Loads libesg_b200.so; raises if it is missing (no fallback path)."""
    global _lib_handle
    if _lib_handle is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C csrc)")
        L = C.CDLL(LIB_PATH)
        L.esg_last_error.restype = C.c_char_p
        L.esg_model_param_count.restype = C.c_int64
        L.esg_model_param_hash.restype = C.c_uint64
        L.esg_adam_lr.restype = C.c_double
        _lib_handle = L
    return _lib_handle


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(rc: int) -> None:
    if rc != OK:
        msg = lib().esg_last_error().decode()
        raise _ERRORS.get(rc, EsgError)(msg)


# --------------------------------------------------------------- structures
@dataclasses.dataclass
class AtomicStructure:
    """structures::AtomicStructure (structure.h:12-36): rows of `cell` are the
    lattice vectors, positions are Cartesian."""

    positions: np.ndarray  # (n, 3) float64
    species: np.ndarray  # (n,) int32 atomic numbers
    cell: np.ndarray  # (3, 3) float64
    pbc: np.ndarray  # (3,) bool

    @property
    def n_atoms(self) -> int:
        return int(self.positions.shape[0])

    def _pbc8(self) -> np.ndarray:
        return np.ascontiguousarray(self.pbc, dtype=np.uint8)


def make_jittered_lattice(n_atoms: int, spacing: float, jitter: float, species_cycle: Sequence[int],
                          seed: int) -> AtomicStructure:
    """model::make_jittered_lattice (synthetic.cpp:17-41)."""
    cyc = np.ascontiguousarray(species_cycle, dtype=np.int32)
    pos = np.zeros((n_atoms, 3))
    cell = np.zeros(9)
    sp = np.zeros(n_atoms, dtype=np.int32)
    _check(lib().esg_jittered_lattice(C.c_int(n_atoms), C.c_double(spacing), C.c_double(jitter), C.c_int(len(cyc)),
                                      _p(cyc), C.c_uint64(seed), _p(pos), _p(cell), _p(sp)))
    return AtomicStructure(pos, sp, cell.reshape(3, 3), np.ones(3, dtype=bool))


def tile(s: AtomicStructure, reps: Sequence[int]) -> AtomicStructure:
    """structures::tile (structure.cpp:40-63)."""
    r = np.ascontiguousarray(reps, dtype=np.int32)
    n = s.n_atoms * int(np.prod(r))
    pos = np.zeros((n, 3))
    cell = np.zeros(9)
    sp = np.zeros(n, dtype=np.int32)
    _check(lib().esg_tile(C.c_int(s.n_atoms), _p(np.ascontiguousarray(s.positions)), _p(np.ascontiguousarray(s.cell)),
                          _p(s._pbc8()), _p(np.ascontiguousarray(s.species, dtype=np.int32)), _p(r), _p(pos), _p(cell),
                          _p(sp)))
    return AtomicStructure(pos, sp, cell.reshape(3, 3), np.array(s.pbc, dtype=bool))


def read_extxyz(path: str) -> AtomicStructure:
    """structures::read_extxyz_file (extxyz.h:17)."""
    n = C.c_int64()
    _check(lib().esg_extxyz_read(path.encode(), C.byref(n), None, None, None, None))
    pos = np.zeros((n.value, 3))
    sp = np.zeros(n.value, dtype=np.int32)
    cell = np.zeros(9)
    pbc = np.zeros(3, dtype=np.uint8)
    _check(lib().esg_extxyz_read(path.encode(), C.byref(n), _p(pos), _p(sp), _p(cell), _p(pbc)))
    return AtomicStructure(pos, sp, cell.reshape(3, 3), pbc.astype(bool))


def write_extxyz(path: str, s: AtomicStructure) -> None:
    """structures::write_extxyz_file (extxyz.h:20)."""
    _check(lib().esg_extxyz_write(path.encode(), C.c_int64(s.n_atoms), _p(np.ascontiguousarray(s.positions)),
                                  _p(np.ascontiguousarray(s.species, dtype=np.int32)),
                                  _p(np.ascontiguousarray(s.cell, dtype=np.float64)), _p(s._pbc8())))


def wrap_positions(s: AtomicStructure) -> np.ndarray:
    """AtomicStructure::wrap (structure.cpp:26-38) on a copy of the positions."""
    pos = np.ascontiguousarray(s.positions, dtype=np.float64).copy()
    _check(lib().esg_wrap_positions(C.c_int(s.n_atoms), _p(pos), _p(np.ascontiguousarray(s.cell)), _p(s._pbc8())))
    return pos


# ------------------------------------------------------------------ context
def nccl_unique_id() -> bytes:
    n = lib().esg_nccl_unique_id_size()
    buf = (C.c_char * n)()
    _check(lib().esg_nccl_get_unique_id(buf))
    return bytes(buf)


class Context:
    """One GPU (and, for world > 1, one NCCL rank)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None):
        self._h = C.c_void_p()
        idbuf = None
        if nccl_id is not None:
            idbuf = (C.c_char * len(nccl_id)).from_buffer_copy(nccl_id)
        _check(lib().esg_ctx_create(C.c_int(device), C.c_int(rank), C.c_int(world), idbuf, C.byref(self._h)))
        self.device, self.rank, self.world = device, rank, world

    def synchronize(self) -> None:
        _check(lib().esg_ctx_synchronize(self._h))

    def close(self) -> None:
        if self._h:
            lib().esg_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# -------------------------------------------------------------------- graph
class Graph:
    """structures::Graph built by esg_build_graph (graph.h:22-37)."""

    def __init__(self, ctx: Context, s: AtomicStructure, r_cut: float):
        self.ctx = ctx
        self._h = C.c_void_p()
        _check(lib().esg_build_graph(ctx._h, C.c_int(s.n_atoms), _p(np.ascontiguousarray(s.positions, np.float64)),
                                     _p(np.ascontiguousarray(s.cell, np.float64)), _p(s._pbc8()), C.c_double(r_cut),
                                     C.byref(self._h)))
        n = C.c_int()
        e = C.c_int64()
        _check(lib().esg_graph_info(self._h, C.byref(n), C.byref(e)))
        self.n_nodes, self.n_edges = n.value, e.value

    def export(self) -> Dict[str, np.ndarray]:
        E = self.n_edges
        out = dict(src=np.zeros(E, np.int32), dst=np.zeros(E, np.int32), shift=np.zeros((E, 3), np.int32),
                   disp=np.zeros((E, 3)), dist=np.zeros(E))
        _check(lib().esg_graph_export(self._h, _p(out["src"]), _p(out["dst"]), _p(out["shift"]), _p(out["disp"]),
                                      _p(out["dist"])))
        return out

    def in_degrees(self) -> np.ndarray:
        d = np.zeros(self.n_nodes, np.int32)
        _check(lib().esg_graph_in_degrees(self._h, _p(d)))
        return d

    def offsets(self) -> np.ndarray:
        o = np.zeros(self.n_nodes + 1, np.int64)
        _check(lib().esg_graph_offsets(self._h, _p(o)))
        return o

    def close(self) -> None:
        if self._h:
            lib().esg_graph_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_graph(ctx: Context, s: AtomicStructure, r_cut: float) -> Graph:
    return Graph(ctx, s, r_cut)


def coupling_matrix(la: int, lb: int, L: int) -> np.ndarray:
    """harmonics::coupling_matrix (clebsch_gordan.h:19)."""
    out = np.zeros((2 * L + 1) * (2 * la + 1) * (2 * lb + 1))
    _check(lib().esg_coupling_matrix(C.c_int(la), C.c_int(lb), C.c_int(L), _p(out)))
    return out.reshape(2 * L + 1, -1)


def lownn_partition(s: AtomicStructure, in_degrees: np.ndarray, depth: int, r_cut: float) -> np.ndarray:
    """partition::lownn_partition (partition.h:24); positions are the unwrapped input."""
    part = np.zeros(s.n_atoms, np.int32)
    _check(lib().esg_lownn_partition(C.c_int(s.n_atoms), _p(np.ascontiguousarray(s.positions, np.float64)),
                                     _p(np.ascontiguousarray(s.cell, np.float64)), _p(s._pbc8()),
                                     _p(np.ascontiguousarray(in_degrees, np.int32)), C.c_int(depth),
                                     C.c_double(r_cut), _p(part)))
    return part


def lownn_partition_gpu(ctx: "Context", s: AtomicStructure, in_degrees: np.ndarray, depth: int,
                        r_cut: float) -> np.ndarray:
    """lownn_partition computed on ctx's device (lownn_gpu.cu); same assignment bit for bit."""
    part = np.zeros(s.n_atoms, np.int32)
    _check(lib().esg_lownn_partition_gpu(ctx._h, C.c_int(s.n_atoms),
                                         _p(np.ascontiguousarray(s.positions, np.float64)),
                                         _p(np.ascontiguousarray(s.cell, np.float64)), _p(s._pbc8()),
                                         _p(np.ascontiguousarray(in_degrees, np.int32)), C.c_int(depth),
                                         C.c_double(r_cut), _p(part)))
    return part


def edge_rotations(ctx: "Context", disp: np.ndarray, l_max: int) -> np.ndarray:
    """build_edge_rotations (kernels.h:43-68) on ctx's device: per edge the
    stacked Wigner blocks D_0..D_lmax (row-major, stride sum (2l+1)^2) of
    align_to_y of the fp32-rounded displacement, as the message kernels
    compute them in-register."""
    d = np.ascontiguousarray(disp, np.float64).reshape(-1, 3)
    ds = (l_max + 1) * (4 * (l_max + 1) ** 2 - 1) // 3
    out = np.zeros((d.shape[0], ds), np.float32)
    _check(lib().esg_edge_rotations(ctx._h, C.c_int64(d.shape[0]), _p(d), C.c_int(l_max), _p(out)))
    return out


class CommPlan:
    """runtime::CommPlan (comm_plan.h:15-35)."""

    def __init__(self, g: Optional[Graph], species: np.ndarray, part: np.ndarray, n_parts: int, rank: int,
                 csr: Optional[tuple] = None):
        """From a device graph, or (csr=(dst_off, src)) from host arrays."""
        self._h = C.c_void_p()
        self._species = np.ascontiguousarray(species, np.int32)
        part = np.ascontiguousarray(part, np.int32)
        if g is not None:
            _check(lib().esg_plan_build(g._h, _p(self._species), _p(part), C.c_int(n_parts), C.c_int(rank),
                                        C.byref(self._h)))
        else:
            off = np.ascontiguousarray(csr[0], np.int64)
            src = np.ascontiguousarray(csr[1], np.int32)
            _check(lib().esg_plan_build_host(C.c_int(len(off) - 1), _p(off), _p(src), _p(self._species), _p(part),
                                             C.c_int(n_parts), C.c_int(rank), C.byref(self._h)))
        info = np.zeros(5, np.int64)
        _check(lib().esg_plan_info(self._h, _p(info)))
        self.n_rows, self.n_owned, self.n_edges, self.n_neighbors, self.n_send = (int(x) for x in info)
        self.rank, self.world = rank, n_parts

    def export(self) -> Dict[str, np.ndarray]:
        z = lambda n: np.zeros(n, np.int32)
        o = dict(row_global=z(self.n_rows), row_species=z(self.n_rows), edge_index=z(self.n_edges),
                 src_row=z(self.n_edges), dst_row=z(self.n_edges), nbr_peer=z(self.n_neighbors),
                 nbr_recv_row=z(self.n_neighbors), nbr_recv_count=z(self.n_neighbors),
                 nbr_send_count=z(self.n_neighbors), send_rows=z(self.n_send))
        _check(lib().esg_plan_export(self._h, *[_p(o[k]) for k in ("row_global", "row_species", "edge_index",
                                                                   "src_row", "dst_row", "nbr_peer",
                                                                   "nbr_recv_row", "nbr_recv_count",
                                                                   "nbr_send_count", "send_rows")]))
        return o

    def close(self) -> None:
        if self._h:
            lib().esg_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_comm_plan(g: Graph, species, part, n_parts: int, rank: int) -> CommPlan:
    return CommPlan(g, species, part, n_parts, rank)


# -------------------------------------------------------------------- model
@dataclasses.dataclass
class ModelConfig:
    """model::ModelConfig (network.h:16-35) + the linear precision knob."""

    l_max: int = 2
    e_width: int = 8
    layers: int = 2
    n_radial: int = 32
    r_cut: float = 4.0
    seed: int = 1
    gate_enabled: bool = True
    linear_precision: int = LINEAR_FP32


@dataclasses.dataclass
class Timing:
    forward_ms: float
    message_ms: float
    halo_ms: float
    heads_ms: float
    exchanges: int
    gpu_launches: int
    halo_skew_ms: float = -1.0
    halo_exchange_ms: float = 0.0
    halo_bytes: int = 0


# ------------------------------------------------------------ input side
def _metrics_from(m, ps, vol):
    parts = np.array([[p.nodes, p.edges, p.neighbors, p.recv_volume] for p in ps], np.int64)
    return Metrics(m.node_imbalance, m.edge_imbalance, m.mean_neighbors, m.max_neighbors, m.total_recv,
                   m.cut_edges, parts, vol, m, ps)


# ------------------------------------------------------- partition metrics
class _PartStats(C.Structure):
    _fields_ = [("nodes", C.c_int64), ("edges", C.c_int64), ("recv_volume", C.c_int64), ("neighbors", C.c_int32),
                ("pad", C.c_int32)]


class _Metrics(C.Structure):
    _fields_ = [("node_imbalance", C.c_double), ("edge_imbalance", C.c_double), ("mean_neighbors", C.c_double),
                ("total_recv", C.c_int64), ("cut_edges", C.c_int64), ("max_neighbors", C.c_int32),
                ("n_parts", C.c_int32)]


@dataclasses.dataclass
class Metrics:
    """partition::Metrics (partition.h:38-46) plus write_dot's volume matrix."""

    node_imbalance: float
    edge_imbalance: float
    mean_neighbors: float
    max_neighbors: int
    total_recv: int
    cut_edges: int
    parts: np.ndarray  # (P, 4) int64: nodes, edges, neighbors, recv_volume
    volume: np.ndarray  # (P, P) int64, [from, to]
    _m: object = None
    _p: object = None

    def json(self) -> str:
        """metrics_json (nlohmann dump(2) format)."""
        n = C.c_int64()
        _check(lib().esg_metrics_json(C.byref(self._m), self._p, None, C.c_int64(0), C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib().esg_metrics_json(C.byref(self._m), self._p, buf, C.c_int64(len(buf)), C.byref(n)))
        return buf.value.decode()

    def dot(self) -> str:
        """write_dot text."""
        P = len(self.parts)
        v = np.ascontiguousarray(self.volume, np.int64)
        n = C.c_int64()
        _check(lib().esg_partition_dot(_p(v), self._p, C.c_int(P), None, C.c_int64(0), C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        _check(lib().esg_partition_dot(_p(v), self._p, C.c_int(P), buf, C.c_int64(len(buf)), C.byref(n)))
        return buf.value.decode()



def partition_metrics(g: "Graph", node_to_part: np.ndarray, n_parts: int) -> Metrics:
    """partition::compute_metrics (metrics.cpp:49-88) on the device."""
    part = np.ascontiguousarray(node_to_part, np.int32)
    if part.size != g.n_nodes:
        raise UsageError(f"assignment covers {part.size} nodes, graph has {g.n_nodes}")
    m = _Metrics()
    ps = (_PartStats * n_parts)()
    vol = np.zeros((n_parts, n_parts), np.int64)
    _check(lib().esg_partition_metrics(g._h, _p(part), C.c_int(n_parts), C.byref(m), ps, _p(vol)))
    return _metrics_from(m, ps, vol)


def metrics_from_arrays(d, i, parts, volume) -> Metrics:
    """A Metrics value from plain numbers (for the host-side formatters)."""
    P = len(parts)
    m = _Metrics(float(d[0]), float(d[1]), float(d[2]), int(i[1]), int(i[2]), int(i[0]), P)
    ps = (_PartStats * P)()
    for q in range(P):
        ps[q].nodes, ps[q].edges, ps[q].neighbors, ps[q].recv_volume = (int(x) for x in parts[q])
    return _metrics_from(m, ps, np.ascontiguousarray(volume, np.int64))


def write_assignment(path: str, node_to_part: np.ndarray) -> None:
    part = np.ascontiguousarray(node_to_part, np.int32)
    _check(lib().esg_assignment_write(os.fsencode(path), _p(part), C.c_int64(part.size)))


def read_assignment(path: str):
    """(node_to_part, n_parts) from a write_assignment file."""
    n, np_ = C.c_int64(), C.c_int()
    _check(lib().esg_assignment_read(os.fsencode(path), None, C.c_int64(0), C.byref(n), C.byref(np_)))
    out = np.zeros(n.value, np.int32)
    _check(lib().esg_assignment_read(os.fsencode(path), _p(out), C.c_int64(out.size), C.byref(n), C.byref(np_)))
    return out, np_.value


# ------------------------------------------------------------- block export
BLOCKS_COUPLED, BLOCKS_UNCOUPLED = 0, 1
BLOCK_KEY = np.dtype([("i", "<i4"), ("j", "<i4"), ("ix", "<i4"), ("iy", "<i4"), ("iz", "<i4"),
                      ("rows", "<u2"), ("cols", "<u2")])  # esg_block_key, 24 bytes
SHARD_HEADER = np.dtype([("magic", "S8"), ("version", "<u4"), ("basis", "<u4"), ("value_bytes", "<u4"),
                         ("flags", "<u4"), ("rank", "<u4"), ("world", "<u4"), ("n_blocks", "<u8"),
                         ("n_values", "<u8"), ("keys_offset", "<u8"), ("values_offset", "<u8")])


def _block_arrays(keys, vals):
    k = np.stack([keys["i"], keys["j"], keys["ix"], keys["iy"], keys["iz"]], axis=1)
    shp = np.stack([keys["rows"], keys["cols"]], axis=1).astype(np.int64)
    off = np.zeros(len(keys) + 1, np.int64)
    np.cumsum(shp[:, 0] * shp[:, 1], out=off[1:])
    return k, shp, off, vals


def read_block_shard(path: str):
    """A shard file memory-mapped: (header dict, keys (n, 5),
    shapes (n, 2), value offsets (n + 1), values)."""
    h = np.fromfile(path, SHARD_HEADER, 1)
    if h.size != 1 or h["magic"][0] != b"ESGBLKS1" or int(h["version"][0]) != 1:
        raise DataError(f"not a block shard: {path}")
    hd = {k: (h[k][0].item() if k != "magic" else h[k][0]) for k in SHARD_HEADER.names}
    nb, nv = hd["n_blocks"], hd["n_values"]
    keys = np.memmap(path, BLOCK_KEY, "r", hd["keys_offset"], (nb,)) if nb else np.zeros(0, BLOCK_KEY)
    vt = np.float64 if hd["value_bytes"] == 8 else np.float32
    vals = np.memmap(path, vt, "r", hd["values_offset"], (nv,)) if nv else np.zeros(0, vt)
    return (hd,) + _block_arrays(keys, vals)


def read_blocks_text(path: str):
    """block_matrix.cpp read_blocks_file: (keys (n, 5), shapes (n, 2), value
    offsets (n + 1), fp64 values), blocks in BlockKey order."""
    nb, nv = C.c_int64(), C.c_int64()
    _check(lib().esg_blocks_read_text(os.fsencode(path), C.byref(nb), C.byref(nv), None, None))
    keys = np.zeros(nb.value, BLOCK_KEY)
    vals = np.zeros(nv.value)
    _check(lib().esg_blocks_read_text(os.fsencode(path), C.byref(nb), C.byref(nv), _p(keys), _p(vals)))
    return _block_arrays(keys, vals)


def merge_block_shards_to_text(shard_paths: Sequence[str], out_path: str) -> None:
    """model_run's rank-0 text file (block_matrix.cpp:90-101) from shards."""
    arr = (C.c_char_p * len(shard_paths))(*[os.fsencode(p) for p in shard_paths])
    _check(lib().esg_blocks_merge_text(arr, C.c_int(len(shard_paths)), os.fsencode(out_path)))


class Network:
    """model::Network<float> (network.h:77-228) driven through the C ABI."""

    def __init__(self, ctx: Optional[Context], cfg: ModelConfig, basis: Dict[int, List[int]]):
        """ctx=None gives a host-only model (parameters, layouts, hash)."""
        self.ctx, self.cfg = ctx, cfg
        zs = sorted(basis)
        z = np.array(zs, np.int32)
        ns = np.array([len(basis[k]) for k in zs], np.int32)
        sh = np.array([l for k in zs for l in basis[k]], np.int32)
        c = _ModelConfig(cfg.l_max, cfg.e_width, cfg.layers, cfg.n_radial, cfg.r_cut, cfg.seed,
                         int(cfg.gate_enabled), cfg.linear_precision)
        self._h = C.c_void_p()
        _check(lib().esg_model_create(ctx._h if ctx is not None else None, C.byref(c), C.c_int(len(z)), _p(z), _p(ns), _p(sh), C.byref(self._h)))
        self.out_len = lib().esg_model_out_len(self._h)
        self.n_params = lib().esg_model_param_count(self._h)

    def set_precision(self, prec: int) -> None:
        _check(lib().esg_model_set_precision(self._h, C.c_int(prec)))
        self.cfg.linear_precision = prec

    def init_params(self) -> None:
        _check(lib().esg_model_init_params(self._h))

    def entries(self):
        out = []
        for i in range(lib().esg_model_n_entries(self._h)):
            name = C.c_char_p()
            r, c, off = C.c_int(), C.c_int(), C.c_int64()
            _check(lib().esg_model_entry(self._h, C.c_int(i), C.byref(name), C.byref(r), C.byref(c), C.byref(off)))
            out.append((name.value.decode(), r.value, c.value, off.value))
        return out

    def params(self) -> np.ndarray:
        p = np.zeros(self.n_params, np.float32)
        _check(lib().esg_model_get_params(self._h, _p(p)))
        return p

    def set_params(self, p: np.ndarray) -> None:
        p = np.ascontiguousarray(p, np.float32)
        assert p.size == self.n_params
        _check(lib().esg_model_set_params(self._h, _p(p)))

    def param_hash(self) -> int:
        return int(lib().esg_model_param_hash(self._h))

    def prepare(self, g: Graph, species: np.ndarray, plan: Optional[CommPlan] = None) -> None:
        sp = np.ascontiguousarray(species, np.int32)
        _check(lib().esg_prepare(self._h, g._h, plan._h if plan is not None else None, _p(sp)))
        info = np.zeros(3, np.int64)
        _check(lib().esg_prepared_info(self._h, _p(info)))
        self.n_rows, self.n_owned, self.n_edges = (int(x) for x in info)

    # ---- training (config 5) ---------------------------------------------
    def set_targets(self, node_target, node_mask, edge_target, edge_mask) -> None:
        """Head-space loss targets of the prepared view (Network::build_targets)."""
        nt = np.ascontiguousarray(node_target, np.float32)
        nm = np.ascontiguousarray(node_mask, np.uint8)
        et = np.ascontiguousarray(edge_target, np.float32)
        em = np.ascontiguousarray(edge_mask, np.uint8)
        assert nt.size == self.n_owned * self.out_len and et.size == self.n_edges * self.out_len
        _check(lib().esg_set_targets(self._h, _p(nt), _p(nm), _p(et), _p(em)))

    def loss_grad(self, n_total: int):
        """Loss (all ranks), this rank's partials and the rank-summed gradients."""
        partials = np.zeros(3)
        loss = C.c_double()
        g = np.zeros(self.n_params, np.float32)
        _check(lib().esg_loss_grad(self._h, C.c_int64(n_total), _p(partials), C.byref(loss), _p(g)))
        return loss.value, partials, g

    def train_step(self, opt: "Adam", n_total: int):
        """DistributedRunner::train_step; returns (loss, forward_ms, backward_ms)."""
        loss = C.c_double()
        t = _Timing()
        _check(lib().esg_train_step(self._h, opt._h, C.c_int64(n_total), C.byref(loss), C.byref(t)))
        return loss.value, t.forward_ms, t.message_ms

    def forward(self, copy_out: bool = True):
        t = _Timing()
        no = eo = None
        if copy_out and hasattr(self, "n_owned"):
            no = np.zeros((self.n_owned, self.out_len), np.float32)
            eo = np.zeros((self.n_edges, self.out_len), np.float32)
        _check(lib().esg_forward(self._h, _p(no), _p(eo), C.byref(t)))
        return no, eo, Timing(t.forward_ms, t.message_ms, t.halo_ms, t.heads_ms, t.exchanges, t.gpu_launches, t.halo_skew_ms,
                      t.halo_exchange_ms, t.halo_bytes)

    def forward_into(self, node_out: Optional[np.ndarray], edge_out: Optional[np.ndarray]) -> Timing:
        """Forward with caller-owned (ideally pinned) host output buffers."""
        t = _Timing()
        _check(lib().esg_forward(self._h, _p(node_out), _p(edge_out), C.byref(t)))
        return Timing(t.forward_ms, t.message_ms, t.halo_ms, t.heads_ms, t.exchanges, t.gpu_launches, t.halo_skew_ms,
                      t.halo_exchange_ms, t.halo_bytes)

    def forward_into_async(self, node_out: Optional[np.ndarray], edge_out: Optional[np.ndarray],
                           timing: bool = True) -> Optional[Timing]:
        """esg_forward_async: with pinned buffers returns once the copies are
        queued; call wait_outputs() before reading or reusing the buffers.
        timing=False: returns as soon as the forward is queued (no Timing)."""
        if not timing:
            _check(lib().esg_forward_async(self._h, _p(node_out), _p(edge_out), None))
            return None
        t = _Timing()
        _check(lib().esg_forward_async(self._h, _p(node_out), _p(edge_out), C.byref(t)))
        return Timing(t.forward_ms, t.message_ms, t.halo_ms, t.heads_ms, t.exchanges, t.gpu_launches, t.halo_skew_ms,
                      t.halo_exchange_ms, t.halo_bytes)

    def wait_outputs(self) -> None:
        _check(lib().esg_forward_wait(self._h))

    def device_outputs(self):
        ptrs = [C.c_void_p() for _ in range(4)]
        _check(lib().esg_forward_outputs(self._h, *[C.byref(p) for p in ptrs]))
        return [p.value for p in ptrs]

    def features(self):
        H = (self.cfg.l_max + 1) ** 2
        n = np.zeros((self.n_rows, H, self.cfg.e_width), np.float32)
        e = np.zeros((self.n_edges, H, self.cfg.e_width), np.float32)
        _check(lib().esg_features_export(self._h, _p(n), _p(e)))
        return n, e

    def outputs_host(self, n_edges: int):
        """Node head outputs and the first n_edges edge head outputs of the
        last forward (esg_outputs_export)."""
        no = np.empty((self.n_owned, self.out_len), np.float32)
        eo = np.empty((n_edges, self.out_len), np.float32)
        _check(lib().esg_outputs_export(self._h, C.c_int64(0), C.c_int64(self.n_owned), _p(no), C.c_int64(0),
                                        C.c_int64(n_edges), _p(eo)))
        return no, eo

    def blocks_uncoupled(self) -> np.ndarray:
        n = C.c_int64()
        _check(lib().esg_blocks_size(self._h, C.byref(n)))
        out = np.zeros(n.value)
        _check(lib().esg_blocks_uncoupled(self._h, _p(out)))
        return out

    def blocks_count(self):
        nb, nv = C.c_int64(), C.c_int64()
        _check(lib().esg_blocks_count(self._h, C.byref(nb), C.byref(nv)))
        return nb.value, nv.value

    def blocks(self, basis: int = 1, symmetrize_onsite: bool = False):
        """This rank's blocks of the last forward: (keys (n, 5) int32 =
        (i, j, ix, iy, iz), shapes (n, 2), value offsets (n + 1), fp64 values)."""
        nb, nv = self.blocks_count()
        keys = np.zeros(nb, BLOCK_KEY)
        vals = np.zeros(nv)
        _check(lib().esg_blocks_export(self._h, C.c_int(basis), C.c_int(int(symmetrize_onsite)), _p(keys), _p(vals)))
        return _block_arrays(keys, vals)

    def build_targets(self, keys: np.ndarray, shapes: np.ndarray, values: np.ndarray):
        """Network::build_targets: uncoupled target blocks (keys (n, 5), shapes
        (n, 2), concatenated row-major values) -> (node_target, node_mask,
        edge_target, edge_mask, count) in head space, view order."""
        n = len(keys)
        rec = np.zeros(n, BLOCK_KEY)
        k = np.asarray(keys).reshape(-1, 5)
        for f, col in zip(("i", "j", "ix", "iy", "iz"), k.T):
            rec[f] = col
        rec["rows"], rec["cols"] = np.asarray(shapes).reshape(-1, 2).T
        v = np.ascontiguousarray(values, np.float64)
        nt = np.zeros((self.n_owned, self.out_len), np.float32)
        nm = np.zeros((self.n_owned, self.out_len), np.uint8)
        et = np.zeros((self.n_edges, self.out_len), np.float32)
        em = np.zeros((self.n_edges, self.out_len), np.uint8)
        cnt = C.c_int64()
        _check(lib().esg_build_targets(self._h, C.c_int64(n), _p(rec), _p(v), _p(nt), _p(nm), _p(et), _p(em),
                                       C.byref(cnt)))
        return nt, nm, et, em, cnt.value

    def blocks_to_device(self, d_keys: int, d_values: int, basis: int = 1, symmetrize_onsite: bool = False,
                         value_bytes: int = 8) -> float:
        """Keys/values into caller device buffers (raw pointers, 0 = skip);
        returns the kernels' device milliseconds."""
        ms = C.c_float()
        _check(lib().esg_blocks_export_device(self._h, C.c_int(basis), C.c_int(int(symmetrize_onsite)),
                                              C.c_int(value_bytes), C.c_void_p(d_keys or None),
                                              C.c_void_p(d_values or None), C.byref(ms)))
        return ms.value

    def write_block_shard(self, path: str, basis: int = 1, symmetrize_onsite: bool = False,
                          value_bytes: int = 8) -> None:
        _check(lib().esg_blocks_write_shard(self._h, os.fsencode(path), C.c_int(basis),
                                            C.c_int(int(symmetrize_onsite)), C.c_int(value_bytes)))

    def write_blocks_text(self, path: str, basis: int = 1, symmetrize_onsite: bool = False) -> None:
        _check(lib().esg_blocks_write_text(self._h, os.fsencode(path), C.c_int(basis),
                                           C.c_int(int(symmetrize_onsite))))

    def save_checkpoint(self, path: str, opt: Optional["Adam"] = None, config_text: str = "") -> None:
        """checkpoint.h save_checkpoint (version-1 container); with opt the
        optimizer section (step, lr, plateau state, fp64 moments) follows."""
        _check(lib().esg_checkpoint_save(self._h, opt._h if opt is not None else None,
                                         config_text.encode(), os.fsencode(path)))

    def load_checkpoint(self, path: str, opt: Optional["Adam"] = None) -> str:
        """checkpoint.h load_checkpoint; restores opt too when given. Returns the config text."""
        buf = C.create_string_buffer(1 << 16)
        _check(lib().esg_checkpoint_load(self._h, opt._h if opt is not None else None,
                                         os.fsencode(path), buf, C.c_int64(len(buf))))
        return buf.value.decode()

    def close(self) -> None:
        if self._h:
            lib().esg_model_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _AdamConfig(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("patience", C.c_int), ("factor", C.c_double), ("threshold", C.c_double), ("min_lr", C.c_double)]


class Adam:
    """model::Optimizer (optimizer.h): Adam, fp64 moments, reduce-on-plateau."""

    def __init__(self, net: Network, **overrides):
        cfg = _AdamConfig()
        lib().esg_adam_default_config(C.byref(cfg))
        for k, v in overrides.items():
            setattr(cfg, k, v)
        self._h = C.c_void_p()
        _check(lib().esg_adam_create(net._h, C.byref(cfg), C.byref(self._h)))

    @property
    def lr(self) -> float:
        return float(lib().esg_adam_lr(self._h))

    def apply(self, net: Network, grads: np.ndarray, loss: float) -> None:
        """Optimizer::step with given gradients (optimizer.h:42-72)."""
        g = np.ascontiguousarray(grads, np.float32)
        assert g.size == net.n_params
        _check(lib().esg_adam_apply(self._h, net._h, _p(g), C.c_double(loss)))

    def close(self) -> None:
        if self._h:
            lib().esg_adam_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------- benchmark configs
# SURVEY.md §8 "Config shorthand": l_max 4, E 16, 32 Gaussians, seed 1.
SI, HF, O = 14, 72, 8
BASIS_SI = {SI: [0, 0, 1, 1, 2]}
BASIS_HFO2 = {HF: [0, 0, 1, 2], O: [0, 1]}


def config_structure(name: str) -> tuple:
    """Returns (structure, r_cut, layers, basis) for C1..C4."""
    if name == "C1":
        return make_jittered_lattice(512, 2.71, 0.30, [SI], 1), 8.0, 1, BASIS_SI
    if name == "C2":
        return make_jittered_lattice(3000, 2.20, 0.45, [HF, O, O], 2), 12.0, 3, BASIS_HFO2
    if name == "C3":
        return make_jittered_lattice(20000, 2.20, 0.45, [HF, O, O], 3), 12.0, 3, BASIS_HFO2
    if name == "C4":
        c2 = make_jittered_lattice(3000, 2.20, 0.45, [HF, O, O], 2)
        return tile(c2, [4, 4, 4]), 10.0, 3, BASIS_HFO2
    raise ValueError(name)
