"""ctypes binding to the REFERENCE implementation compiled as the oracle's pin
(oracle/_ref/libesgnn_ref.so, built by oracle/ref.mk from /root/reference
sources against oracle/eigen_shim; test infrastructure only).

available() is False when the library was not built (no /root/reference
where build() ran); the tests that need it skip then.
"""
import ctypes as C
import os
from typing import Dict, List, Optional

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB_PATH = os.path.join(ROOT, "oracle", "_ref", "libesgnn_ref.so")
ACCEPTANCE = os.path.join(ROOT, "oracle", "_ref", "ref_acceptance")
_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_build_graph.restype = C.c_int64
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _ok(rc):
    if rc != 0:
        raise RuntimeError(lib().ref_last_error().decode())


def jittered_lattice(n, spacing, jitter, cycle, seed):
    pos = np.zeros((n, 3))
    cell = np.zeros((3, 3))
    sp = np.zeros(n, np.int32)
    cyc = np.asarray(cycle, np.int32)
    _ok(lib().ref_jittered_lattice(C.c_int(n), C.c_double(spacing), C.c_double(jitter), C.c_int(len(cyc)), _p(cyc),
                                   C.c_uint64(seed), _p(pos), _p(cell), _p(sp)))
    return pos, cell, sp


_keep = []  # converted inputs stay alive until the next call


def _struct_args(pos, species, cell, pbc):
    arrs = [np.ascontiguousarray(pos, np.float64), np.ascontiguousarray(species, np.int32),
            np.ascontiguousarray(cell, np.float64), np.ascontiguousarray(pbc, np.uint8)]
    _keep[:] = arrs
    return (C.c_int(len(pos)),) + tuple(_p(a) for a in arrs)


def build_graph(pos, species, cell, pbc, r_cut) -> Dict[str, np.ndarray]:
    args = _struct_args(pos, species, cell, pbc)
    E = lib().ref_build_graph(*args, C.c_double(r_cut))
    if E < 0:
        raise RuntimeError(lib().ref_last_error().decode())
    g = dict(src=np.zeros(E, np.int32), dst=np.zeros(E, np.int32), shift=np.zeros((E, 3), np.int32),
             disp=np.zeros((E, 3)), dist=np.zeros(E))
    lib().ref_graph_export(_p(g["src"]), _p(g["dst"]), _p(g["shift"]), _p(g["disp"]), _p(g["dist"]))
    return g


def lownn(pos, species, cell, pbc, depth, r_cut) -> np.ndarray:
    """On the graph of the last build_graph call."""
    part = np.zeros(len(pos), np.int32)
    _ok(lib().ref_lownn(*_struct_args(pos, species, cell, pbc), C.c_int(depth), C.c_double(r_cut), _p(part)))
    return part


def comm_plan(species, part, n_parts, rank) -> Dict[str, np.ndarray]:
    """On the graph of the last build_graph call."""
    sp = np.ascontiguousarray(species, np.int32)
    pt = np.ascontiguousarray(part, np.int32)
    info = np.zeros(5, np.int64)
    _ok(lib().ref_comm_plan(_p(sp), C.c_int(n_parts), _p(pt), C.c_int(rank), _p(info), None, None, None, None, None,
                            None, None))
    n_rows, n_owned, ne, nn, ns = (int(x) for x in info)
    z = lambda n: np.zeros(n, np.int32)
    o = dict(row_global=z(n_rows), src_row=z(ne), dst_row=z(ne), nbr_peer=z(nn), nbr_recv_row=z(nn),
             nbr_recv_count=z(nn), send_rows=z(ns))
    _ok(lib().ref_comm_plan(_p(sp), C.c_int(n_parts), _p(pt), C.c_int(rank), _p(info), _p(o["row_global"]),
                            _p(o["src_row"]), _p(o["dst_row"]), _p(o["nbr_peer"]), _p(o["nbr_recv_row"]),
                            _p(o["nbr_recv_count"]), _p(o["send_rows"])))
    o["n_owned"] = n_owned
    return o


def _basis_args(basis: Dict[int, List[int]]):
    zs = sorted(basis)
    z = np.array(zs, np.int32)
    ns = np.array([len(basis[k]) for k in zs], np.int32)
    sh = np.array([l for k in zs for l in basis[k]], np.int32)
    return (C.c_int(len(zs)), _p(z), _p(ns), _p(sh)), (z, ns, sh)


def out_len(basis) -> int:
    args, keep = _basis_args(basis)
    n = lib().ref_out_len(*args)
    if n < 0:
        raise RuntimeError(lib().ref_last_error().decode())
    return n


def forward(pos, species, cell, pbc, r_cut, basis, l_max=4, e_width=16, layers=1, n_radial=32, seed=1, gate=True,
            precision=4, coupled_path: Optional[str] = None, uncoupled_path: Optional[str] = None):
    """The reference's taped Network<T> forward on the serial view
    (network.h:115-164): node heads (n x out_len) and edge heads (E x
    out_len, the reference edge order), as float64 arrays."""
    g = build_graph(pos, species, cell, pbc, r_cut)
    ol = out_len(basis)
    no = np.zeros((len(pos), ol))
    eo = np.zeros((len(g["src"]), ol))
    bargs, keep = _basis_args(basis)
    _ok(lib().ref_forward(*_struct_args(pos, species, cell, pbc), C.c_double(r_cut), *bargs, C.c_int(l_max),
                          C.c_int(e_width), C.c_int(layers), C.c_int(n_radial), C.c_uint64(seed), C.c_int(int(gate)),
                          C.c_int(precision), _p(no), _p(eo),
                          coupled_path.encode() if coupled_path else None,
                          uncoupled_path.encode() if uncoupled_path else None))
    return no, eo, g


def forward_view_timed(view, basis, layers, r_cut, threads, l_max=4, e_width=16, n_radial=32, seed=1):
    """The reference's Network<float>::prepare + build_forward on a view
    (dict as oracle.serial_view / bench.cpu_sample build it), the owned
    destinations split over `threads` threads.  Returns (prepare s, forward s),
    each the max over threads."""
    arrs = [np.ascontiguousarray(view["row_species"], np.int32), np.ascontiguousarray(view["src_row"], np.int32),
            np.ascontiguousarray(view["dst_row"], np.int32), np.ascontiguousarray(view["disp"], np.float64),
            np.ascontiguousarray(view["dist"], np.float64)]
    bargs, keep = _basis_args(basis)
    secs = np.zeros(2)
    _ok(lib().ref_forward_view_timed(C.c_int(int(view["n_rows"])), C.c_int(int(view["n_owned"])), _p(arrs[0]),
                                     C.c_int64(len(arrs[1])), _p(arrs[1]), _p(arrs[2]), _p(arrs[3]), _p(arrs[4]),
                                     *bargs, C.c_int(l_max), C.c_int(e_width), C.c_int(layers), C.c_int(n_radial),
                                     C.c_double(r_cut), C.c_uint64(seed), C.c_int(threads), _p(secs)))
    return float(secs[0]), float(secs[1])


def read_extxyz(path):
    """structures::read_extxyz_file: (positions, species, cell, pbc)."""
    n = C.c_int64()
    _ok(lib().ref_read_extxyz(path.encode(), C.byref(n), None, None, None, None))
    pos = np.zeros((n.value, 3))
    sp = np.zeros(n.value, np.int32)
    cell = np.zeros((3, 3))
    pbc = np.zeros(3, np.uint8)
    _ok(lib().ref_read_extxyz(path.encode(), C.byref(n), _p(pos), _p(sp), _p(cell), _p(pbc)))
    return pos, sp, cell, pbc


def write_extxyz(path, pos, species, cell, pbc):
    args = _struct_args(pos, species, cell, pbc)
    _ok(lib().ref_write_extxyz(path.encode(), *args))
