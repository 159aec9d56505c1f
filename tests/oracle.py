"""ctypes wrapper of oracle/liboracle.so -- the CPU restatement of the
reference (test infrastructure: only tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline legs may use it, and only as the checker)."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, List

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
_L = None


def lib() -> C.CDLL:
    global _L
    if _L is None:
        if not os.path.exists(ORACLE_SO):
            subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], check=True, capture_output=True)
        L = C.CDLL(ORACLE_SO)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_build_graph.restype = C.c_int64
        L.oracle_face_spacing.restype = C.c_double
        L.oracle_model_create.restype = C.c_void_p
        L.oracle_model_param_count.restype = C.c_int64
        L.oracle_model_entry.restype = C.c_char_p
        for f in ("oracle_model_destroy", "oracle_model_out_len", "oracle_model_n_entries",
                  "oracle_model_params_f32", "oracle_model_params_f64", "oracle_model_set_params_f32",
                  "oracle_forward_f32", "oracle_forward_f64", "oracle_uncoupled_block", "oracle_model_param_count",
                  "oracle_model_entry", "oracle_backward_f32", "oracle_backward_f64", "oracle_toy_targets",
                  "oracle_model_set_params_f64"):
            getattr(L, f).argtypes = None
        _L = L
    return _L


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _ok(rc):
    if rc != 0:
        raise RuntimeError(lib().oracle_last_error().decode())


def set_threads(n: int) -> None:
    lib().oracle_set_threads(C.c_int(n))


def num_threads() -> int:
    return lib().oracle_num_threads()


def jittered_lattice(n, spacing, jitter, cycle, seed):
    cyc = np.ascontiguousarray(cycle, np.int32)
    pos = np.zeros((n, 3))
    cell = np.zeros(9)
    sp = np.zeros(n, np.int32)
    _ok(lib().oracle_jittered_lattice(C.c_int(n), C.c_double(spacing), C.c_double(jitter), C.c_int(len(cyc)), _p(cyc),
                                      C.c_uint64(seed), _p(pos), _p(cell), _p(sp)))
    return pos, cell.reshape(3, 3), sp


def tile(pos, cell, pbc, species, reps):
    n = pos.shape[0] * int(np.prod(reps))
    po = np.zeros((n, 3))
    co = np.zeros(9)
    so = np.zeros(n, np.int32)
    _ok(lib().oracle_tile(C.c_int(pos.shape[0]), _p(np.ascontiguousarray(pos)), _p(np.ascontiguousarray(cell)),
                          _p(np.ascontiguousarray(pbc, np.uint8)), _p(np.ascontiguousarray(species, np.int32)),
                          _p(np.ascontiguousarray(reps, np.int32)), _p(po), _p(co), _p(so)))
    return po, co.reshape(3, 3), so


def wrap(pos, cell, pbc):
    p = np.ascontiguousarray(pos, np.float64).copy()
    _ok(lib().oracle_wrap(C.c_int(p.shape[0]), _p(p), _p(np.ascontiguousarray(cell)),
                          _p(np.ascontiguousarray(pbc, np.uint8))))
    return p


def face_spacing(cell, d):
    return lib().oracle_face_spacing(_p(np.ascontiguousarray(cell, np.float64)), C.c_int(d))


def build_graph(pos, cell, pbc, r_cut) -> Dict[str, np.ndarray]:
    E = lib().oracle_build_graph(C.c_int(pos.shape[0]), _p(np.ascontiguousarray(pos, np.float64)),
                                 _p(np.ascontiguousarray(cell, np.float64)), _p(np.ascontiguousarray(pbc, np.uint8)),
                                 C.c_double(r_cut))
    if E < 0:
        raise RuntimeError(lib().oracle_last_error().decode())
    g = dict(src=np.zeros(E, np.int32), dst=np.zeros(E, np.int32), shift=np.zeros((E, 3), np.int32),
             disp=np.zeros((E, 3)), dist=np.zeros(E))
    lib().oracle_graph_export(_p(g["src"]), _p(g["dst"]), _p(g["shift"]), _p(g["disp"]), _p(g["dist"]))
    return g


def in_degrees(n, g):
    return np.bincount(g["dst"], minlength=n).astype(np.int32)


def lownn(pos, cell, pbc, deg, depth, r_cut):
    out = np.zeros(pos.shape[0], np.int32)
    _ok(lib().oracle_lownn(C.c_int(pos.shape[0]), _p(np.ascontiguousarray(pos, np.float64)),
                           _p(np.ascontiguousarray(cell, np.float64)), _p(np.ascontiguousarray(pbc, np.uint8)),
                           _p(np.ascontiguousarray(deg, np.int32)), C.c_int(depth), C.c_double(r_cut), _p(out)))
    return out


def compute_metrics(n, src, dst, part, P):
    """metrics.cpp:49-88: (parts (P, 4) nodes/edges/neighbors/recv_volume,
    (node_imbalance, edge_imbalance, mean_neighbors), (max_neighbors,
    total_recv, cut_edges))."""
    parts = np.zeros((P, 4), np.int64)
    d = np.zeros(3)
    i = np.zeros(3, np.int64)
    _ok(lib().oracle_compute_metrics(C.c_int(n), C.c_int64(len(src)), _p(np.ascontiguousarray(src, np.int32)),
                                     _p(np.ascontiguousarray(dst, np.int32)), _p(np.ascontiguousarray(part, np.int32)),
                                     C.c_int(P), _p(parts), _p(d), _p(i)))
    return parts, d, i


def write_dot(n, src, dst, part, P, path):
    """metrics.cpp:141-166."""
    _ok(lib().oracle_write_dot(C.c_int(n), C.c_int64(len(src)), _p(np.ascontiguousarray(src, np.int32)),
                               _p(np.ascontiguousarray(dst, np.int32)), _p(np.ascontiguousarray(part, np.int32)),
                               C.c_int(P), os.fsencode(str(path))))


def nlohmann_double(v):
    """nlohmann::json's double output (dtoa_impl::to_chars + format_buffer,
    min_exp -4, max_exp 15), restated; shortest round-trip digits from repr."""
    import math
    if not math.isfinite(v):
        return "null"
    sign = "-" if math.copysign(1.0, v) < 0 else ""
    v = abs(v)
    if v == 0.0:
        return sign + "0.0"
    r = repr(v)
    if "e" in r:
        m, e = r.split("e")
        digits, n = m.replace(".", ""), int(e) + 1
    else:
        ip, fp = r.split(".")
        if ip != "0":
            digits, n = (ip + fp).rstrip("0") or "0", len(ip)
        else:
            z = len(fp) - len(fp.lstrip("0"))
            digits, n = fp.lstrip("0"), -z
    digits = digits.lstrip("0") or "0"
    k = len(digits)
    if k <= n <= 15:
        return sign + digits + "0" * (n - k) + ".0"
    if 0 < n <= 15:
        return sign + digits[:n] + "." + digits[n:]
    if -4 < n <= 0:
        return sign + "0." + "0" * (-n) + digits
    m = digits[0] + ("." + digits[1:] if k > 1 else "")
    e = n - 1
    return sign + m + "e" + ("-" if e < 0 else "+") + f"{abs(e):02d}"


def nlohmann_dump2(obj, indent=0):
    """nlohmann::json::dump(2): std::map key order, ': ' and ',\n'."""
    pad, inner = " " * indent, " " * (indent + 2)
    if isinstance(obj, dict):
        if not obj:
            return "{}"
        items = [f'{inner}"{k}": {nlohmann_dump2(obj[k], indent + 2)}' for k in sorted(obj)]
        return "{\n" + ",\n".join(items) + "\n" + pad + "}"
    if isinstance(obj, list):
        if not obj:
            return "[]"
        return "[\n" + ",\n".join(inner + nlohmann_dump2(x, indent + 2) for x in obj) + "\n" + pad + "]"
    if isinstance(obj, float):
        return nlohmann_double(obj)
    return str(int(obj))


def metrics_json(parts, d, i):
    """metrics.cpp:124-139 metrics_json."""
    return nlohmann_dump2({
        "n_parts": len(parts), "node_imbalance": float(d[0]), "edge_imbalance": float(d[1]),
        "mean_neighbors": float(d[2]), "max_neighbors": int(i[0]), "total_recv_volume": int(i[1]),
        "cut_edges": int(i[2]),
        "parts": [{"nodes": int(p[0]), "edges": int(p[1]), "neighbors": int(p[2]), "recv_volume": int(p[3])}
                  for p in parts]})


def comm_plan(n_nodes, src, dst, part, n_parts, rank):
    E = len(src)
    hdr = np.zeros(4, np.int32)
    rg = np.zeros(n_nodes, np.int32)
    ei = np.zeros(E, np.int32)
    sr = np.zeros(E, np.int32)
    dr = np.zeros(E, np.int32)
    peer = np.zeros(n_parts, np.int32)
    rr = np.zeros(n_parts, np.int32)
    rc = np.zeros(n_parts, np.int32)
    sc = np.zeros(n_parts, np.int32)
    rows = np.zeros(E + n_nodes, np.int32)
    _ok(lib().oracle_comm_plan(C.c_int(n_nodes), C.c_int64(E), _p(np.ascontiguousarray(src, np.int32)),
                               _p(np.ascontiguousarray(dst, np.int32)), _p(np.ascontiguousarray(part, np.int32)),
                               C.c_int(n_parts), C.c_int(rank), _p(hdr), _p(rg), _p(ei), _p(sr), _p(dr), _p(peer),
                               _p(rr), _p(rc), _p(sc), _p(rows)))
    n_rows, n_owned, ne, nn = (int(x) for x in hdr)
    return dict(n_rows=n_rows, n_owned=n_owned, row_global=rg[:n_rows], edge_index=ei[:ne], src_row=sr[:ne],
                dst_row=dr[:ne], nbr_peer=peer[:nn], nbr_recv_row=rr[:nn], nbr_recv_count=rc[:nn],
                nbr_send_count=sc[:nn], send_rows=rows[:int(sc[:nn].sum())])


def align_wigner(r, l_max):
    R = np.zeros(9)
    n = sum((2 * l + 1) ** 2 for l in range(l_max + 1))
    D = np.zeros(n)
    lib().oracle_align_wigner(_p(np.ascontiguousarray(r, np.float64)), C.c_int(l_max), _p(R), _p(D))
    return R.reshape(3, 3), split_blocks(D, l_max)


def wigner(R, l_max):
    n = sum((2 * l + 1) ** 2 for l in range(l_max + 1))
    D = np.zeros(n)
    lib().oracle_wigner(_p(np.ascontiguousarray(R, np.float64)), C.c_int(l_max), _p(D))
    return split_blocks(D, l_max)


def split_blocks(D, l_max) -> List[np.ndarray]:
    out, o = [], 0
    for l in range(l_max + 1):
        d = 2 * l + 1
        out.append(D[o:o + d * d].reshape(d, d))
        o += d * d
    return out


def real_sh(r, l_max):
    y = np.zeros((l_max + 1) ** 2)
    lib().oracle_real_sh(_p(np.ascontiguousarray(r, np.float64)), C.c_int(l_max), _p(y))
    return y


def coupling(la, lb, L):
    out = np.zeros((2 * L + 1) * (2 * la + 1) * (2 * lb + 1))
    _ok(lib().oracle_coupling(C.c_int(la), C.c_int(lb), C.c_int(L), _p(out)))
    return out.reshape(2 * L + 1, (2 * la + 1) * (2 * lb + 1))


def m_layout(l_max):
    h = (l_max + 1) ** 2
    to_m = np.zeros(h, np.int32)
    to_l = np.zeros(h, np.int32)
    mo = np.zeros(l_max + 1, np.int32)
    lib().oracle_m_layout(C.c_int(l_max), _p(to_m), _p(to_l), _p(mo))
    return to_m, to_l, mo


class Model:
    """Network<T> restatement: config + basis + seeded ParamStore."""

    def __init__(self, l_max, e_width, layers, n_radial, r_cut, seed, basis: Dict[int, List[int]], gate=True):
        zs = sorted(basis)
        z = np.array(zs, np.int32)
        ns = np.array([len(basis[k]) for k in zs], np.int32)
        sh = np.array([l for k in zs for l in basis[k]], np.int32)
        L = lib()
        self.h = L.oracle_model_create(C.c_int(l_max), C.c_int(e_width), C.c_int(layers), C.c_int(n_radial),
                                       C.c_double(r_cut), C.c_uint64(seed), C.c_int(int(gate)), C.c_int(len(z)), _p(z),
                                       _p(ns), _p(sh))
        if not self.h:
            raise RuntimeError(L.oracle_last_error().decode())
        self.l_max, self.e, self.layers = l_max, e_width, layers
        self.H = (l_max + 1) ** 2
        self.out_len = L.oracle_model_out_len(C.c_void_p(self.h))
        self.n_params = L.oracle_model_param_count(C.c_void_p(self.h))

    def __del__(self):
        try:
            lib().oracle_model_destroy(C.c_void_p(self.h))
        except Exception:
            pass

    def entries(self):
        out = []
        for i in range(lib().oracle_model_n_entries(C.c_void_p(self.h))):
            r, c, off = C.c_int(), C.c_int(), C.c_int64()
            name = lib().oracle_model_entry(C.c_void_p(self.h), C.c_int(i), C.byref(r), C.byref(c), C.byref(off))
            out.append((name.decode(), r.value, c.value, off.value))
        return out

    def params_f32(self):
        p = np.zeros(self.n_params, np.float32)
        lib().oracle_model_params_f32(C.c_void_p(self.h), _p(p))
        return p

    def params_f64(self):
        p = np.zeros(self.n_params, np.float64)
        lib().oracle_model_params_f64(C.c_void_p(self.h), _p(p))
        return p

    def set_params_f32(self, p):
        lib().oracle_model_set_params_f32(C.c_void_p(self.h), _p(np.ascontiguousarray(p, np.float32)))

    def _call(self, dtype, view, mode, nodes=None, edges=None, layer=0, node_block=0, node_out=None, edge_out=None):
        f = lib().oracle_forward_f32 if dtype == np.float32 else lib().oracle_forward_f64
        E = len(view["src_row"])
        _ok(f(C.c_void_p(self.h), C.c_int(view["n_rows"]), C.c_int(view["n_owned"]),
              _p(np.ascontiguousarray(view["row_species"], np.int32)), C.c_int64(E),
              _p(np.ascontiguousarray(view["src_row"], np.int32)), _p(np.ascontiguousarray(view["dst_row"], np.int32)),
              _p(np.ascontiguousarray(view["disp"], np.float64)), _p(np.ascontiguousarray(view["dist"], np.float64)),
              C.c_int(mode), _p(nodes), _p(edges), C.c_int(layer), C.c_int(node_block), _p(node_out), _p(edge_out)))

    def forward(self, view, dtype=np.float32, features=False):
        """Serial forward (mode 0).  Returns node_out, edge_out[, nodes, edges]."""
        E = len(view["src_row"])
        no = np.zeros((view["n_owned"], self.out_len), dtype)
        eo = np.zeros((E, self.out_len), dtype)
        nodes = np.zeros((view["n_rows"], self.H, self.e), dtype) if features else None
        edges = np.zeros((E, self.H, self.e), dtype) if features else None
        self._call(dtype, view, 0, nodes, edges, node_out=no, edge_out=eo)
        return (no, eo, nodes, edges) if features else (no, eo)

    def init_tables(self, view, dtype=np.float32):
        E = len(view["src_row"])
        nodes = np.zeros((view["n_rows"], self.H, self.e), dtype)
        edges = np.zeros((E, self.H, self.e), dtype)
        self._call(dtype, view, 1, nodes, edges)
        return nodes, edges

    def block(self, view, nodes, edges, layer, node_block):
        self._call(nodes.dtype.type, view, 2, nodes, edges, layer=layer, node_block=int(node_block))

    def heads(self, view, nodes, edges):
        E = len(view["src_row"])
        no = np.zeros((view["n_owned"], self.out_len), nodes.dtype)
        eo = np.zeros((E, self.out_len), nodes.dtype)
        self._call(nodes.dtype.type, view, 3, nodes, edges, node_out=no, edge_out=eo)
        return no, eo

    def set_params_f64(self, p):
        lib().oracle_model_set_params_f64(C.c_void_p(self.h), _p(np.ascontiguousarray(p, np.float64)))

    def _bwd(self, view, mode, nodes, edges, layer=0, node_block=0, g_node_out=None, g_edge_out=None, g_nodes=None,
             g_edges=None, grads=None):
        dt = grads.dtype.type
        f = lib().oracle_backward_f32 if dt == np.float32 else lib().oracle_backward_f64
        E = len(view["src_row"])
        _ok(f(C.c_void_p(self.h), C.c_int(view["n_rows"]), C.c_int(view["n_owned"]),
              _p(np.ascontiguousarray(view["row_species"], np.int32)), C.c_int64(E),
              _p(np.ascontiguousarray(view["src_row"], np.int32)), _p(np.ascontiguousarray(view["dst_row"], np.int32)),
              _p(np.ascontiguousarray(view["disp"], np.float64)), _p(np.ascontiguousarray(view["dist"], np.float64)),
              C.c_int(mode), _p(nodes), _p(edges), C.c_int(layer), C.c_int(int(node_block)), _p(g_node_out),
              _p(g_edge_out), _p(g_nodes), _p(g_edges), _p(grads)))

    def block_backward(self, view, nodes, edges, layer, node_block, g_nodes, g_edges, grads):
        """ops.h backward closures of one block; g_nodes/g_edges: output grads in, input grads out."""
        self._bwd(view, 0, nodes, edges, layer, node_block, g_nodes=g_nodes, g_edges=g_edges, grads=grads)

    def heads_backward(self, view, nodes, edges, g_node_out, g_edge_out, g_nodes, g_edges, grads):
        self._bwd(view, 1, nodes, edges, g_node_out=g_node_out, g_edge_out=g_edge_out, g_nodes=g_nodes,
                  g_edges=g_edges, grads=grads)

    def init_backward(self, view, g_nodes, g_edges, grads):
        self._bwd(view, 2, None, None, g_nodes=g_nodes, g_edges=g_edges, grads=grads)

    def toy_targets(self, n, species, g):
        """synthetic.cpp toy_hamiltonian encoded into head space (serial view,
        graph-edge order): (node_t, node_m, edge_t, edge_m, node_t64, edge_t64)."""
        E = len(g["src"])
        nt = np.zeros((n, self.out_len), np.float32)
        nm = np.zeros((n, self.out_len), np.uint8)
        et = np.zeros((E, self.out_len), np.float32)
        em = np.zeros((E, self.out_len), np.uint8)
        nt64 = np.zeros((n, self.out_len))
        et64 = np.zeros((E, self.out_len))
        _ok(lib().oracle_toy_targets(C.c_void_p(self.h), C.c_int(n), _p(np.ascontiguousarray(species, np.int32)),
                                      C.c_int64(E), _p(np.ascontiguousarray(g["src"], np.int32)),
                                      _p(np.ascontiguousarray(g["dst"], np.int32)),
                                      _p(np.ascontiguousarray(g["shift"], np.int32)),
                                      _p(np.ascontiguousarray(g["disp"], np.float64)),
                                      _p(np.ascontiguousarray(g["dist"], np.float64)), _p(nt), _p(nm), _p(nt64), _p(et),
                                      _p(em), _p(et64)))
        return nt, nm, et, em, nt64, et64

    def uncoupled_block(self, za, zb, row, n_orb_a, n_orb_b):
        out = np.zeros(n_orb_a * n_orb_b)
        _ok(lib().oracle_uncoupled_block(C.c_void_p(self.h), C.c_int(za), C.c_int(zb),
                                         _p(np.ascontiguousarray(row, np.float32)), _p(out)))
        return out.reshape(n_orb_a, n_orb_b)

    def export_text(self, keys, rows, species, coupled_path, uncoupled_path):
        """model_run.cpp:141-153 for one rank: coupled map, its text,
        blocks_to_uncoupled, its text (the block export's CPU baseline)."""
        k = np.ascontiguousarray(keys, np.int32)
        r = np.ascontiguousarray(rows, np.float32)
        _ok(lib().oracle_export_text(C.c_void_p(self.h), C.c_int64(len(k)), _p(k), _p(r), C.c_int(r.shape[1]),
                                     _p(np.ascontiguousarray(species, np.int32)), os.fsencode(str(coupled_path)),
                                     os.fsencode(str(uncoupled_path))))

    def coupled_block(self, za, zb, row, n_orb_a, n_orb_b):
        """network.h:296-315 fill_block."""
        out = np.zeros(n_orb_a * n_orb_b)
        _ok(lib().oracle_coupled_block(C.c_void_p(self.h), C.c_int(za), C.c_int(zb),
                                       _p(np.ascontiguousarray(row, np.float32)), _p(out)))
        return out.reshape(n_orb_a, n_orb_b)


def write_blocks(keys, shapes, values, path):
    """block_matrix.cpp:90-101 write_blocks (std::ostream, precision 17) of the
    map gather_blocks builds (model_run.cpp:103-120): equal keys keep the last
    block.  keys (n, 5), shapes (n, 2), values concatenated row-major."""
    k7 = np.ascontiguousarray(np.concatenate([np.asarray(keys, np.int32).reshape(-1, 5),
                                              np.asarray(shapes, np.int32).reshape(-1, 2)], axis=1))
    v = np.ascontiguousarray(values, np.float64)
    _ok(lib().oracle_write_blocks(C.c_int64(len(k7)), _p(k7), _p(v), os.fsencode(str(path))))


def serial_view(n, species, g):
    """model::serial_view (graph_view.h:37-56) as plain arrays."""
    return dict(n_rows=n, n_owned=n, row_species=np.asarray(species, np.int32), src_row=g["src"], dst_row=g["dst"],
                disp=g["disp"], dist=g["dist"])


def plan_view(plan, species, g):
    ei = plan["edge_index"]
    return dict(n_rows=plan["n_rows"], n_owned=plan["n_owned"],
                row_species=np.asarray(species, np.int32)[plan["row_global"]], src_row=plan["src_row"],
                dst_row=plan["dst_row"], disp=g["disp"][ei], dist=g["dist"][ei])


# ------------------------------------------------------------------ training
def masked_loss(pred, target, mask, n_total):
    """ops.h:347-371: partials (sum_abs, sum_sq, count) in fp64 and the seed
    gradient (sign(d) + 2 d) / n_total cast to the prediction's type."""
    d = pred.astype(np.float64) - np.asarray(target, np.float64)
    m = np.asarray(mask, bool)
    sa = float(np.abs(d[m]).sum())
    sq = float((d[m] ** 2).sum())
    g = np.where(m, (np.sign(d) + 2.0 * d) / float(n_total), 0.0).astype(pred.dtype)
    return (sa, sq, int(m.sum())), g


def loss_grad(model, view, targets, n_total, dtype=np.float64, exchange=None, exchange_bwd=None):
    """Network::record_loss + Tape::backward (serial or one rank): returns
    (partials, grads) with grads laid out like the parameters.  exchange /
    exchange_bwd(g_nodes) run around every block for multi-rank drivers."""
    node_t, node_m, edge_t, edge_m = targets
    nodes, edges = model.init_tables(view, dtype)
    saved = []
    for layer in range(model.layers):
        for nb in (True, False):
            if exchange is not None:
                exchange(nodes)
            saved.append((layer, nb, nodes.copy(), edges.copy()))
            model.block(view, nodes, edges, layer, nb)
    no, eo = model.heads(view, nodes, edges)
    pn, gno = masked_loss(no, node_t, node_m, n_total)
    pe, geo = masked_loss(eo, edge_t, edge_m, n_total)
    grads = np.zeros(model.n_params, dtype)
    g_nodes = np.zeros_like(nodes)
    g_edges = np.zeros_like(edges)
    model.heads_backward(view, nodes, edges, np.ascontiguousarray(gno), np.ascontiguousarray(geo), g_nodes, g_edges,
                         grads)
    for layer, nb, n_in, e_in in reversed(saved):
        model.block_backward(view, n_in, e_in, layer, nb, g_nodes, g_edges, grads)
        if exchange_bwd is not None:
            exchange_bwd(g_nodes)
    model.init_backward(view, g_nodes, g_edges, grads)
    return (pn[0] + pe[0], pn[1] + pe[1], pn[2] + pe[2]), grads


class Adam:
    """optimizer.h:15-80 (moments in fp64, reduce-on-plateau)."""

    def __init__(self, n, lr=5e-3, beta1=0.9, beta2=0.999, eps=1e-8, patience=100, factor=0.5, threshold=1e-4,
                 min_lr=1e-6):
        self.m = np.zeros(n)
        self.v = np.zeros(n)
        self.lr, self.b1, self.b2, self.eps = lr, beta1, beta2, eps
        self.patience, self.factor, self.threshold, self.min_lr = patience, factor, threshold, min_lr
        self.t, self.best, self.stale = 0, float("inf"), 0

    def step(self, params, grads, loss):
        self.t += 1
        g = np.asarray(grads, np.float64)
        self.m = self.b1 * self.m + (1.0 - self.b1) * g
        self.v = self.b2 * self.v + (1.0 - self.b2) * g * g
        mh = self.m / (1.0 - self.b1 ** self.t)
        vh = self.v / (1.0 - self.b2 ** self.t)
        out = (params.astype(np.float64) - self.lr * mh / (np.sqrt(vh) + self.eps)).astype(params.dtype)
        if loss < self.best * (1.0 - self.threshold):
            self.best, self.stale = loss, 0
        else:
            self.stale += 1
            if self.stale >= self.patience:
                self.lr = max(self.min_lr, self.lr * self.factor)
                self.stale = 0
        return out


# ------------------------------------------------------------ input side
SYMBOLS = ("", "H", "He", "Li", "Be", "B", "C", "N", "O", "F", "Ne", "Na", "Mg", "Al", "Si", "P", "S", "Cl", "Ar",
           "K", "Ca", "Sc", "Ti", "V", "Cr", "Mn", "Fe", "Co", "Ni", "Cu", "Zn", "Ga", "Ge", "As", "Se", "Br",
           "Kr", "Rb", "Sr", "Y", "Zr", "Nb", "Mo", "Tc", "Ru", "Rh", "Pd", "Ag", "Cd", "In", "Sn", "Sb", "Te",
           "I", "Xe", "Cs", "Ba", "La", "Ce", "Pr", "Nd", "Pm", "Sm", "Eu", "Gd", "Tb", "Dy", "Ho", "Er", "Tm",
           "Yb", "Lu", "Hf", "Ta", "W", "Re", "Os", "Ir", "Pt", "Au", "Hg", "Tl", "Pb", "Bi", "Po", "At", "Rn",
           "Fr", "Ra", "Ac", "Th", "Pa", "U", "Np", "Pu", "Am", "Cm", "Bk", "Cf", "Es", "Fm", "Md", "No",
           "Lr")  # elements.cpp:15-23


class ParseError(ValueError):
    pass


def read_extxyz_text(text):
    """extxyz.cpp:16-121 read_extxyz: (pos (n,3), species, cell (3,3), pbc)."""
    lines = text.split("\n")
    if text.endswith("\n"):
        lines = lines[:-1]
    if not lines:
        raise ParseError("empty input")
    try:
        natoms = int(lines[0].split()[0])
    except (IndexError, ValueError):
        raise ParseError("expected atom count")
    if natoms < 0:
        raise ParseError("expected atom count")
    if len(lines) < 2:
        raise ParseError("missing comment line")
    kv, line, i = {}, lines[1], 0
    while i < len(line):
        while i < len(line) and line[i].isspace():
            i += 1
        if i >= len(line):
            break
        k0 = i
        while i < len(line) and line[i] != "=" and not line[i].isspace():
            i += 1
        if i >= len(line) or line[i] != "=":
            continue
        key = line[k0:i]
        i += 1
        if i < len(line) and line[i] == '"':
            j = line.find('"', i + 1)
            if j < 0:
                raise ParseError("unterminated quote")
            val, i = line[i + 1:j], j + 1
        else:
            j = i
            while j < len(line) and not line[j].isspace():
                j += 1
            val, i = line[i:j], j
        kv[key] = val
    cell, pbc = np.eye(3), np.zeros(3, bool)
    if "Lattice" in kv:
        t = kv["Lattice"].split()
        if len(t) < 9:
            raise ParseError("Lattice needs 9 numbers")
        cell = np.array([float(x) for x in t[:9]]).reshape(3, 3)
        pbc[:] = True
    if "pbc" in kv:
        t = kv["pbc"].split()
        if len(t) < 3:
            raise ParseError("pbc needs 3 flags")
        for d in range(3):
            if t[d] in ("T", "true", "True", "1"):
                pbc[d] = True
            elif t[d] in ("F", "false", "False", "0"):
                pbc[d] = False
            else:
                raise ParseError("bad pbc flag")
    if pbc.any() and "Lattice" not in kv:
        raise ParseError("pbc set but no Lattice given")
    pos, sp = [], []
    for k in range(natoms):
        if 2 + k >= len(lines):
            raise ParseError("fewer atom lines than declared")
        t = lines[2 + k].split()
        if len(t) < 4:
            raise ParseError("expected 'Symbol x y z'")
        if t[0] not in SYMBOLS[1:]:
            raise ValueError("unknown element symbol")
        sp.append(SYMBOLS.index(t[0]))
        pos.append([float(x) for x in t[1:4]])
    return np.array(pos, np.float64).reshape(-1, 3), np.array(sp, np.int32), cell, pbc


def write_extxyz_text(pos, species, cell, pbc):
    """extxyz.cpp:125-140 write_extxyz (std::ostream precision 17 = %.17g)."""
    out = [f"{len(species)}"]
    head = ""
    if any(pbc):
        head = 'Lattice="' + " ".join("%.17g" % x for x in np.asarray(cell).ravel()) + '" pbc="' + \
            " ".join("T" if b else "F" for b in pbc) + '"'
    out.append(head)
    for z, p in zip(species, pos):
        out.append(SYMBOLS[z] + " " + " ".join("%.17g" % x for x in p))
    return "\n".join(out) + "\n"


def _splitmix(x):
    m = (1 << 64) - 1
    x = (x + 0x9e3779b97f4a7c15) & m
    x = ((x ^ (x >> 30)) * 0xbf58476d1ce4e5b9) & m
    x = ((x ^ (x >> 27)) * 0x94d049bb133111eb) & m
    return x ^ (x >> 31)


def mincut(n, dst_off, src, n_parts, seed=1):
    """mincut.cpp:16-201 mincut_partition, pure Python (small graphs)."""
    from collections import deque
    dst = np.repeat(np.arange(n), np.diff(dst_off))
    pairs = sorted((int(s), int(d)) for s, d in zip(src, dst) if s != d)
    adj = [[] for _ in range(n)]  # per source: (nbr, multiplicity) in pair order
    k = 0
    while k < len(pairs):
        j = k
        while j < len(pairs) and pairs[j] == pairs[k]:
            j += 1
        adj[pairs[k][0]].append((pairs[k][1], j - k))
        k = j
    wt = [max(1, int(dst_off[v + 1] - dst_off[v])) for v in range(n)]
    wmax = max(wt) if wt else 1
    out = [0] * n

    def bisect(nodes, np_, base, sd):
        if np_ == 1:
            for v in nodes:
                out[v] = base
            return
        npl, npr, m = (np_ + 1) // 2, np_ // 2, len(nodes)
        local = {v: i for i, v in enumerate(nodes)}
        total = sum(wt[v] for v in nodes)
        target = total * npl // np_
        slack = max(total // 20, wmax)

        def bfs(start):
            order, seen, q, scan = [], [False] * m, deque(), 0
            seen[start] = True
            q.append(start)
            while len(order) < m:
                if not q:
                    while seen[scan]:
                        scan += 1
                    seen[scan] = True
                    q.append(scan)
                v = q.popleft()
                order.append(v)
                for u, _ in adj[nodes[v]]:
                    lu = local.get(u, -1)
                    if lu >= 0 and not seen[lu]:
                        seen[lu] = True
                        q.append(lu)
            return order

        far = bfs(_splitmix(sd) % m)[-1]
        side, lw, taken = [1] * m, 0, 0
        for v in bfs(far):
            if taken >= m - 1 or (lw >= target and taken >= 1):
                break
            side[v], lw, taken = 0, lw + wt[nodes[v]], taken + 1

        def gain_of(v):
            g = 0
            for u, w in adj[nodes[v]]:
                lu = local.get(u, -1)
                if lu >= 0:
                    g += w if side[lu] != side[v] else -w
            return g

        for _ in range(8):
            gain = [gain_of(v) for v in range(m)]
            locked, moves, run, best, best_len, cur = [False] * m, [], 0, 0, 0, lw
            for _step in range(m):
                pick = -1
                for v in range(m):
                    if locked[v]:
                        continue
                    after = cur - wt[nodes[v]] if side[v] == 0 else cur + wt[nodes[v]]
                    if abs(after - target) > slack:
                        continue
                    if pick < 0 or gain[v] > gain[pick]:
                        pick = v
                if pick < 0:
                    break
                run += gain[pick]
                cur += -wt[nodes[pick]] if side[pick] == 0 else wt[nodes[pick]]
                side[pick] ^= 1
                locked[pick] = True
                moves.append(pick)
                gain[pick] = -gain[pick]
                for u, w in adj[nodes[pick]]:
                    lu = local.get(u, -1)
                    if lu < 0 or locked[lu]:
                        continue
                    gain[lu] += -2 * w if side[lu] == side[pick] else 2 * w
                if run > best:
                    best, best_len = run, len(moves)
            for v in reversed(moves[best_len:]):
                side[v] ^= 1
            lw = sum(wt[nodes[v]] for v in range(m) if side[v] == 0)
            if best <= 0:
                break
        left = [nodes[v] for v in range(m) if side[v] == 0]
        right = [nodes[v] for v in range(m) if side[v] == 1]
        if len(left) < npl or len(right) < npr:
            cut = min(max(m * npl // np_, npl), m - npr)
            left, right = nodes[:cut], nodes[cut:]
        bisect(left, npl, base, _splitmix(sd ^ 0x51ed2701))
        bisect(right, npr, base + npl, _splitmix(sd ^ 0xa24baed4))

    if n_parts < 1 or n_parts > max(1, n):
        raise ValueError("bad part count")
    if n_parts > 1 and n > 0:
        bisect(list(range(n)), n_parts, 0, seed)
    return np.array(out, np.int32)
