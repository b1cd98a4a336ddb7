"""Thin ctypes binding of libspa.so (include/spa.h).  Argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; there is no CPU or
PyTorch fallback: if libspa.so is missing, importing anything that needs it raises.
PyTorch is used only for device memory, streams and process groups (tensors are passed
to the library as raw pointers + element strides).

The same names as the C ABI are exported (spa_kv_alloc, spa_kv_append, ...), plus small
convenience classes (Pool, Plan, Comm, Peer) that own the handles.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SPA_LIB: a variant build (libspa_NAME.so next to this file, build.py --variant) for
# performance experiments; the default is the library build() produces
LIB_PATH = os.path.join(HERE, os.path.basename(os.environ.get("SPA_LIB", "libspa.so")))

SPA_OK, SPA_ERR_INVALID_ARG, SPA_ERR_NO_PAGES, SPA_ERR_BAD_REQUEST = 0, 1, 2, 3
SPA_ERR_CUDA, SPA_ERR_NCCL, SPA_ERR_UNSUPPORTED, SPA_ERR_NO_DEVICE, SPA_ERR_WORKSPACE = 4, 5, 6, 7, 8

c_int32, c_int64, c_void_p, c_float = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_float
P_int32 = ctypes.POINTER(c_int32)
P_int64 = ctypes.POINTER(c_int64)


class SpaError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"spa status {status}: {message}")
        self.status = status
        self.message = message


class spa_pool_config(ctypes.Structure):
    _fields_ = [("num_layers", c_int32), ("num_q_heads", c_int32), ("num_kv_heads", c_int32),
                ("head_dim", c_int32), ("page_size", c_int32), ("num_pages", c_int32)]


class spa_plan_config(ctypes.Structure):
    _fields_ = [("sharing", c_int32), ("max_rows", c_int32), ("split_pages", c_int32), ("num_ctas", c_int32),
                ("merge_mode", c_int32), ("teams_per_cta", c_int32)]


class spa_plan_stats(ctypes.Structure):
    _fields_ = [("n_req", c_int32), ("n_groups", c_int32), ("n_desc", c_int32), ("n_items", c_int32),
                ("n_records", c_int32), ("n_teams", c_int32), ("rows_max", c_int32), ("generation", c_int32),
                ("unique_tokens", c_int64), ("unshared_tokens", c_int64), ("pages_read", c_int64),
                ("alg_tokens", c_int64)]


# name -> (restype, argtypes); mirrors include/spa.h and include/spa_debug.h
_SIGS = {
    "spa_pool_create": (c_int32, [ctypes.POINTER(spa_pool_config), c_void_p, c_void_p, ctypes.POINTER(c_void_p)]),
    "spa_pool_destroy": (c_int32, [c_void_p]),
    "spa_pool_create_fp8": (c_int32, [ctypes.POINTER(spa_pool_config), c_void_p, c_void_p, ctypes.POINTER(c_void_p)]),
    "spa_kv_alloc": (c_int32, [c_void_p, P_int64]),
    "spa_kv_append": (c_int32, [c_void_p, c_int32, P_int64, P_int32, c_void_p, c_void_p, c_void_p]),
    "spa_fork_request": (c_int32, [c_void_p, c_int64, c_int32, P_int64, c_void_p]),
    "spa_kv_free": (c_int32, [c_void_p, c_int64]),
    "spa_kv_release_window": (c_int32, [c_void_p, c_int32, P_int64, c_int32]),
    "spa_kv_page_table": (c_int32, [c_void_p, c_int64, P_int32, c_int32, P_int32, P_int32]),
    "spa_pool_refcounts": (c_int32, [c_void_p, P_int32]),
    "spa_pool_free_pages": (c_int32, [c_void_p, P_int32, c_int32, P_int32]),
    "spa_plan_create": (c_int32, [c_void_p, ctypes.POINTER(spa_plan_config), ctypes.POINTER(c_void_p)]),
    "spa_plan_destroy": (c_int32, [c_void_p]),
    "spa_decode_plan": (c_int32, [c_void_p, c_int32, P_int64, c_int32, c_void_p]),
    "spa_extend_plan": (c_int32, [c_void_p, c_int32, P_int64, P_int32, c_int32, c_void_p]),
    "spa_plan_get_stats": (c_int32, [c_void_p, ctypes.POINTER(spa_plan_stats)]),
    "spa_plan_set_workspace": (c_int32, [c_void_p, c_void_p, ctypes.c_size_t]),
    "spa_plan_workspace_size": (c_int32, [c_void_p, ctypes.POINTER(ctypes.c_size_t)]),
    "spa_decode_attention": (c_int32, [c_void_p, c_int32, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_int64,
                                       c_void_p, c_int64, c_int64, c_float, c_void_p]),
    "spa_merge_splits": (c_int32, [c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                   c_int64, c_void_p, c_int64, c_int64, c_void_p]),
    "spa_nccl_unique_id": (c_int32, [c_void_p]),
    "spa_comm_create": (c_int32, [c_void_p, c_int32, c_int32, ctypes.POINTER(c_void_p)]),
    "spa_comm_destroy": (c_int32, [c_void_p]),
    "spa_decode_attention_sharded": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_int64, c_int64, c_void_p,
                                               c_void_p, c_float, c_void_p]),
    "spa_peer_create": (c_int32, [c_int32, c_int32, ctypes.c_size_t, c_int32, ctypes.POINTER(c_void_p)]),
    "spa_peer_ipc_handle": (c_int32, [c_void_p, c_void_p]),
    "spa_peer_connect": (c_int32, [c_void_p, c_void_p]),
    "spa_peer_connect_local": (c_int32, [ctypes.POINTER(c_void_p), c_int32]),
    "spa_peer_buffer": (c_int32, [c_void_p, c_int32, ctypes.POINTER(c_void_p)]),
    "spa_peer_status": (c_int32, [c_void_p, P_int32]),
    "spa_peer_destroy": (c_int32, [c_void_p]),
    "spa_decode_attention_fused_gather": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_int64, c_int64, c_int32,
                                                    c_int32, c_float, c_void_p]),
    "spa_abi_version": (c_int32, []),
    "spa_last_error": (ctypes.c_char_p, []),
    "spa_plan_debug_array": (c_int32, [c_void_p, c_int32, ctypes.POINTER(P_int32), P_int64, P_int32]),
    "spa_debug_read_bw_ldg": (c_int32, [c_void_p, ctypes.c_size_t, c_void_p, c_void_p]),
    "spa_debug_pool_read_tma": (c_int32, [c_void_p, c_int32, c_int32, c_void_p]),
    "spa_debug_set_trace": (c_int32, [c_void_p, c_void_p, c_int32]),
    "spa_debug_umma_selftest": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "spa_debug_plan_geometry": (c_int32, [c_void_p, P_int32, P_int32, P_int32]),
}


def read_ceilings(pool: "Pool", scratch_bytes: int = 4 << 30, reps: int = 5, stream=None) -> dict:
    """Same-run read-bandwidth ceilings (GB/s): streaming LDG over a scratch buffer, and the
    decode kernel's TMA pipeline without math over the pool (include/spa_debug.h)."""
    import torch  # noqa: WPS433

    dev = pool.k.device
    buf = torch.empty(scratch_bytes // 2, dtype=torch.bfloat16, device=dev)
    buf.fill_(1.0)
    sink = torch.zeros(4, dtype=torch.int32, device=dev)
    s = _stream_ptr(stream)
    out = {}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    best = 0.0
    for _ in range(reps):
        ev[0].record()
        _check(lib().spa_debug_read_bw_ldg(_ptr(buf), buf.numel() * 2, _ptr(sink), s))
        ev[1].record()
        torch.cuda.synchronize()
        best = max(best, buf.numel() * 2 / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9)
    out["ldg_read_gbs"] = best
    del buf
    if getattr(pool, "fp8", False):   # the TMA probe is bf16-only
        return out
    c = pool.cfg
    per_layer = (c.num_pages // 2 * 2) * c.num_kv_heads * c.page_size * c.head_dim * 2 * 2
    layers = max(1, min(c.num_layers, (8 << 30) // max(1, per_layer)))
    for mode, name in ((0, "tma_pool_read_gbs"), (1, "tma3d_pool_read_gbs"), (2, "bulk_pool_read_gbs")):
        best = 0.0
        for _ in range(reps):
            ev[0].record()
            _check(lib().spa_debug_pool_read_tma(pool.h, layers, mode, s))
            ev[1].record()
            torch.cuda.synchronize()
            best = max(best, layers * per_layer / (ev[0].elapsed_time(ev[1]) * 1e-3) / 1e9)
        out[name] = best
    out["tma_probe_bytes"] = layers * per_layer
    return out

def umma_selftest(q, k, v, stream=None):
    """tcgen05 descriptor/TMEM self-test (include/spa_debug.h): returns (S, O) fp32."""
    import torch  # noqa: WPS433

    s = torch.empty((128, 32), dtype=torch.float32, device=q.device)
    o = torch.empty((128, 128), dtype=torch.float32, device=q.device)
    _check(lib().spa_debug_umma_selftest(_ptr(q), _ptr(k), _ptr(v), _ptr(s), _ptr(o), _stream_ptr(stream)))
    return s, o


_lib = None


def lib() -> ctypes.CDLL:
    """Load libspa.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run `python -m paper_2511_20048_b200.build` "
                               "(there is no CPU fallback)")
        if "SPA_NCCL_LIB" not in os.environ:
            try:
                import nvidia.nccl  # noqa: WPS433
                cand = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
                if os.path.exists(cand):
                    os.environ["SPA_NCCL_LIB"] = cand
            except ImportError:
                pass
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int):
    if status != SPA_OK:
        raise SpaError(status, lib().spa_last_error().decode(errors="replace"))


def _stream_ptr(stream):
    if stream is None:
        import torch  # noqa: WPS433

        if not torch.cuda.is_available():
            return None
        return c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return c_void_p(stream)
    return c_void_p(stream.cuda_stream)


def _ptr(t):
    return None if t is None else c_void_p(t.data_ptr())


# ---------------------------------------------------------------------------- same-name wrappers
def spa_abi_version() -> int:
    return lib().spa_abi_version()


def spa_pool_create(cfg: spa_pool_config, k_pool_ptr, v_pool_ptr):
    h = c_void_p()
    _check(lib().spa_pool_create(ctypes.byref(cfg), k_pool_ptr, v_pool_ptr, ctypes.byref(h)))
    return h


def spa_pool_destroy(h):
    _check(lib().spa_pool_destroy(h))


def spa_kv_alloc(pool_h) -> int:
    r = c_int64()
    _check(lib().spa_kv_alloc(pool_h, ctypes.byref(r)))
    return r.value


def spa_kv_append(pool_h, reqs, n_new, k_new_ptr, v_new_ptr, stream_ptr):
    n = len(reqs)
    ra = (c_int64 * max(n, 1))(*reqs)
    na = (c_int32 * max(n, 1))(*n_new)
    return lib().spa_kv_append(pool_h, n, ra, na, k_new_ptr, v_new_ptr, stream_ptr)


def spa_fork_request(pool_h, parent: int, prefix_len: int, stream_ptr):
    c = c_int64()
    st = lib().spa_fork_request(pool_h, parent, prefix_len, ctypes.byref(c), stream_ptr)
    return st, c.value


def spa_kv_free(pool_h, req: int):
    return lib().spa_kv_free(pool_h, req)


def spa_kv_page_table(pool_h, req: int):
    n = c_int32()
    ln = c_int32()
    st = lib().spa_kv_page_table(pool_h, req, None, 0, ctypes.byref(n), ctypes.byref(ln))
    if st != SPA_OK:
        return st, None, None
    buf = (c_int32 * max(n.value, 1))()
    _check(lib().spa_kv_page_table(pool_h, req, buf, n.value, ctypes.byref(n), ctypes.byref(ln)))
    return st, list(buf[:n.value]), ln.value


# ---------------------------------------------------------------------------- classes
class Pool:
    """A paged KV pool.  device=None -> metadata-only pool (host logic only)."""

    def __init__(self, num_layers, num_q_heads, num_kv_heads, head_dim, num_pages, page_size=16, device=None,
                 kv_scale=None):
        """kv_scale: fp32 [L, Hkv, 2] (k_scale, v_scale) -> an FP8 (e4m3) pool (spa_pool_create_fp8)."""
        self.cfg = spa_pool_config(num_layers, num_q_heads, num_kv_heads, head_dim, page_size, num_pages)
        self.k = self.v = None
        self.fp8 = kv_scale is not None
        self.kv_scale = None
        if device is not None:
            import torch  # noqa: WPS433

            if self.fp8:
                self.kv_scale = torch.as_tensor(kv_scale, dtype=torch.float32).reshape(
                    num_layers, num_kv_heads, 2).to(device).contiguous()
                # one interleaved buffer: per page-head the K block then the transposed V block
                self.kv = torch.empty((num_layers, num_pages, num_kv_heads, 2, page_size, head_dim),
                                      dtype=torch.uint8, device=device)
                self.k = self.kv[:, :, :, 0]                                       # [L, P, Hkv, 16, d]
                self.v = self.kv[:, :, :, 1].view(num_layers, num_pages, num_kv_heads, head_dim, page_size)
            else:
                shape = (num_layers, num_pages, num_kv_heads, page_size, head_dim)
                self.k = torch.empty(shape, dtype=torch.bfloat16, device=device)
                self.v = torch.empty(shape, dtype=torch.bfloat16, device=device)
        if self.fp8:
            h = c_void_p()
            _check(lib().spa_pool_create_fp8(ctypes.byref(self.cfg), _ptr(getattr(self, "kv", None)),
                                             _ptr(self.kv_scale), ctypes.byref(h)))
            self.h = h
        else:
            self.h = spa_pool_create(self.cfg, _ptr(self.k), _ptr(self.v))

    @property
    def num_pages(self):
        return self.cfg.num_pages

    def close(self):
        if self.h:
            spa_pool_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 (interpreter shutdown)
            pass

    def alloc(self) -> int:
        return spa_kv_alloc(self.h)

    def append(self, reqs, n_new, k_new=None, v_new=None, stream=None, check=True):
        """k_new, v_new: bf16 tensors [L, sum(n_new), Hkv, d] (contiguous)."""
        for t in (k_new, v_new):
            if t is not None and not t.is_contiguous():
                raise ValueError("k_new / v_new must be contiguous")
        st = spa_kv_append(self.h, list(reqs), list(n_new), _ptr(k_new), _ptr(v_new),
                           _stream_ptr(stream) if self.k is not None else None)
        if check:
            _check(st)
        return st

    def fork(self, parent, prefix_len, stream=None, check=True):
        st, child = spa_fork_request(self.h, parent, prefix_len, _stream_ptr(stream) if self.k is not None else None)
        if check:
            _check(st)
            return child
        return st, child

    def release_window(self, reqs, window: int, check=True):
        """spa_kv_release_window: drop the pages no future query can read under `window`."""
        arr = (c_int64 * max(1, len(reqs)))(*reqs)
        st = lib().spa_kv_release_window(self.h, len(reqs), arr, int(window))
        if check:
            _check(st)
        return st

    def free(self, req, check=True):
        st = spa_kv_free(self.h, req)
        if check:
            _check(st)
        return st

    def page_table(self, req):
        return spa_kv_page_table(self.h, req)

    def refcounts(self):
        buf = (c_int32 * self.cfg.num_pages)()
        _check(lib().spa_pool_refcounts(self.h, buf))
        return list(buf)

    def free_pages(self):
        n = c_int32()
        buf = (c_int32 * self.cfg.num_pages)()
        _check(lib().spa_pool_free_pages(self.h, buf, self.cfg.num_pages, ctypes.byref(n)))
        return list(buf[:n.value])


class Plan:
    def __init__(self, pool: Pool, sharing=True, max_rows=0, split_pages=0, num_ctas=0, merge_mode=0,
                 teams_per_cta=0, workspace=None):
        """max_rows: 0 auto (16 or 32 rows per item, per batch), 16, 32, 64, 128.
        merge_mode: 0 in-kernel tail phase (default), 1 in-kernel last arriver, 2 merge kernel.
        workspace: a caller-owned uint8 device tensor for the plan (include/spa.h
        spa_plan_set_workspace), fixed; None = a torch tensor this object grows on demand."""
        self.pool = pool
        cfg = spa_plan_config(1 if sharing else 0, max_rows, split_pages, num_ctas, int(merge_mode), int(teams_per_cta))
        h = c_void_p()
        _check(lib().spa_plan_create(pool.h, ctypes.byref(cfg), ctypes.byref(h)))
        self.h = h
        self.n_req = 0
        self._ws = None
        self._ws_fixed = workspace is not None
        if workspace is not None:
            self.set_workspace(workspace)

    def set_workspace(self, ws):
        """Hand the plan a caller-owned device workspace (uint8 tensor, 256-B aligned)."""
        self._ws = ws
        _check(lib().spa_plan_set_workspace(self.h, _ptr(ws), ws.numel() * ws.element_size()))

    def workspace_size(self) -> int:
        n = ctypes.c_size_t()
        _check(lib().spa_plan_workspace_size(self.h, ctypes.byref(n)))
        return n.value

    def close(self):
        if self.h:
            _check(lib().spa_plan_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def plan(self, reqs, window=0, stream=None, check=True, n_query=None):
        """Plan a decode batch (one query row per request), or with n_query (one int per
        request) an extend batch: request i's last n_query[i] tokens are query rows
        (request-major, token-minor), each attending causally (include/spa.h)."""
        n = len(reqs)
        ra = (c_int64 * max(n, 1))(*reqs)
        sp = _stream_ptr(stream) if self.pool.k is not None else None
        if n_query is None:
            st = lib().spa_decode_plan(self.h, n, ra, int(window), sp)
            rows = n
        else:
            if len(n_query) != n:
                raise ValueError("n_query needs one entry per request")
            qa = (c_int32 * max(n, 1))(*[int(x) for x in n_query])
            st = lib().spa_extend_plan(self.h, n, ra, qa, int(window), sp)
            rows = int(sum(int(x) for x in n_query))
        if st == SPA_ERR_WORKSPACE and not self._ws_fixed:
            import torch  # noqa: WPS433

            need = self.workspace_size()
            self.set_workspace(torch.empty(need + need // 2 + 4096, dtype=torch.uint8, device=self.pool.k.device))
            if n_query is None:
                st = lib().spa_decode_plan(self.h, n, ra, int(window), sp)
            else:
                st = lib().spa_extend_plan(self.h, n, ra, qa, int(window), sp)
        if check:
            _check(st)
            self.n_req = rows
        return st

    def stats(self) -> dict:
        s = spa_plan_stats()
        _check(lib().spa_plan_get_stats(self.h, ctypes.byref(s)))
        return {f: getattr(s, f) for f, _ in s._fields_}

    def debug_array(self, which: int):
        data = P_int32()
        n = c_int64()
        w = c_int32()
        _check(lib().spa_plan_debug_array(self.h, which, ctypes.byref(data), ctypes.byref(n), ctypes.byref(w)))
        flat = [data[i] for i in range(n.value)]
        if w.value > 1:
            return [flat[i:i + w.value] for i in range(0, len(flat), w.value)]
        return flat

    def geometry(self) -> tuple:
        """(num_ctas, teams_per_cta, warps_per_cta) of the plan's decode launches."""
        nc, tm, wp = c_int32(), c_int32(), c_int32()
        _check(lib().spa_debug_plan_geometry(self.h, ctypes.byref(nc), ctypes.byref(tm), ctypes.byref(wp)))
        return nc.value, tm.value, wp.value

    def num_ctas_hint(self) -> int:
        nc, tm, wp = c_int32(), c_int32(), c_int32()
        _check(lib().spa_debug_plan_geometry(self.h, ctypes.byref(nc), ctypes.byref(tm), ctypes.byref(wp)))
        return nc.value

    def set_trace(self, cap: int = 0):
        """Timeline trace of the next decode launches (include/spa_debug.h); cap 0 = off.
        Returns the (zeroed) uint64 device buffer [num_ctas * warps_per_cta, cap, 2], or None."""
        import torch  # noqa: WPS433

        if cap <= 0:
            _check(lib().spa_debug_set_trace(self.h, None, 0))
            self._trace = None
            return None
        nc, tm, wp = c_int32(), c_int32(), c_int32()
        _check(lib().spa_debug_plan_geometry(self.h, ctypes.byref(nc), ctypes.byref(tm), ctypes.byref(wp)))
        buf = torch.zeros((nc.value * wp.value, cap, 2), dtype=torch.int64, device=self.pool.k.device)
        _check(lib().spa_debug_set_trace(self.h, _ptr(buf), cap))
        self._trace = buf
        return buf

    def decode(self, layer, q, o=None, lse=None, scale=None, stream=None, want_lse=True):
        """q: bf16 [N, Hq, d] (any strides, d contiguous).  Returns (o, lse)."""
        import torch  # noqa: WPS433

        N, Hq, d = q.shape
        if scale is None:
            scale = d ** -0.5
        if o is None:
            o = torch.empty((N, Hq, d), dtype=torch.bfloat16, device=q.device)
        if lse is None and want_lse:
            lse = torch.empty((N, Hq), dtype=torch.float32, device=q.device)
        if q.stride(2) != 1 or o.stride(2) != 1:
            raise ValueError("head_dim must be contiguous")
        _check(lib().spa_decode_attention(
            self.h, int(layer), _ptr(q), q.stride(0), q.stride(1), _ptr(o), o.stride(0), o.stride(1),
            _ptr(lse), lse.stride(0) if lse is not None else 0, lse.stride(1) if lse is not None else 0,
            float(scale), _stream_ptr(stream)))
        return o, lse

    def decode_sharded(self, comm, layer, q_local, o_gathered, lse_gathered=None, scale=None, stream=None):
        d = q_local.shape[-1]
        if scale is None:
            scale = d ** -0.5
        _check(lib().spa_decode_attention_sharded(
            self.h, comm.h, int(layer), _ptr(q_local), q_local.stride(0), q_local.stride(1),
            _ptr(o_gathered), _ptr(lse_gathered), float(scale), _stream_ptr(stream)))
        return o_gathered, lse_gathered


def spa_merge_splits(rec_ptr, part_o, part_lse, o, lse=None, stream=None):
    """rec_ptr int32 [N+1], part_o fp32 [S, H, d], part_lse fp32 [S, H] (device tensors)."""
    N = rec_ptr.numel() - 1
    S, H, d = part_o.shape
    _check(lib().spa_merge_splits(N, H, d, _ptr(rec_ptr), _ptr(part_o), _ptr(part_lse), _ptr(o), o.stride(0),
                                  o.stride(1), _ptr(lse), lse.stride(0) if lse is not None else 0,
                                  lse.stride(1) if lse is not None else 0, _stream_ptr(stream)))
    return o, lse


def shard_heads(num_q_heads: int, num_kv_heads: int, rank: int, world: int):
    """KV-head sharding: rank r holds KV heads [r Hkv/n, (r+1) Hkv/n)
    and the query heads that read them, [r Hq/n, (r+1) Hq/n) (kv = floor(h / G), reading #5)."""
    if num_kv_heads % world or num_q_heads % num_kv_heads:
        raise ValueError("world must divide num_kv_heads and num_kv_heads must divide num_q_heads")
    hkv, hq = num_kv_heads // world, num_q_heads // world
    return slice(rank * hq, (rank + 1) * hq), slice(rank * hkv, (rank + 1) * hkv)


def spa_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().spa_nccl_unique_id(buf))
    return buf.raw


class Comm:
    def __init__(self, unique_id: bytes, rank: int, world: int):
        h = c_void_p()
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(lib().spa_comm_create(buf, rank, world, ctypes.byref(h)))
        self.h = h
        self.rank, self.world = rank, world

    def close(self):
        if self.h:
            _check(lib().spa_comm_destroy(self.h))
            self.h = None


class _DevArray:
    """A raw device pointer as a __cuda_array_interface__ object (to view library-owned
    memory as a torch tensor without copying)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


class Peer:
    """F1 fused decode + all-gather over peer memory (include/spa.h spa_peer_*).

    Owns this rank's library-allocated region (n_bufs gathered-output buffers + a signal
    pad).  Multi-process: pass the torch.distributed group; the 64-byte CUDA IPC handles
    are all-gathered through it.  Virtual ranks in one process: Peer.local_world()."""

    def __init__(self, rank: int, world: int, buf_bytes: int, n_bufs: int = 2, group=None, connect=True):
        h = c_void_p()
        _check(lib().spa_peer_create(rank, world, int(buf_bytes), n_bufs, ctypes.byref(h)))
        self.h, self.rank, self.world, self.n_bufs, self.buf_bytes = h, rank, world, n_bufs, int(buf_bytes)
        if world > 1 and connect:
            import torch.distributed as dist  # noqa: WPS433

            allh = [None] * world
            dist.all_gather_object(allh, self.ipc_handle(), group=group)
            self.connect(allh)

    def ipc_handle(self) -> bytes:
        """This rank's 64-byte CUDA IPC handle of its region."""
        mine = ctypes.create_string_buffer(64)
        _check(lib().spa_peer_ipc_handle(self.h, mine))
        return mine.raw

    def connect(self, handles):
        """Open every other rank's region (handles in rank order)."""
        blob = ctypes.create_string_buffer(b"".join(handles), 64 * self.world)
        _check(lib().spa_peer_connect(self.h, blob))

    @staticmethod
    def local_world(world: int, buf_bytes: int, n_bufs: int = 2) -> list["Peer"]:
        peers = [Peer(r, world, buf_bytes, n_bufs, connect=False) for r in range(world)]
        arr = (c_void_p * world)(*[p.h.value for p in peers])
        _check(lib().spa_peer_connect_local(arr, world))
        return peers

    @staticmethod
    def buffer_bytes(n_req: int, num_q_heads: int, head_dim: int, with_lse: bool = True) -> int:
        """Bytes of one gathered buffer: O bf16 [Hq][N][d] (+ LSE fp32 [Hq][N] at a 256-B offset)."""
        ob = num_q_heads * n_req * head_dim * 2
        return ((ob + 255) & ~255) + (num_q_heads * n_req * 4 if with_lse else 0)

    def views(self, buf_idx: int, n_req: int, num_q_heads: int, head_dim: int, device=None):
        """(O [Hq][N][d] bf16, LSE [Hq][N] fp32) views of this rank's buffer buf_idx."""
        import torch  # noqa: WPS433

        ptr = c_void_p()
        _check(lib().spa_peer_buffer(self.h, buf_idx, ctypes.byref(ptr)))
        dev = device or torch.device("cuda", torch.cuda.current_device())
        o = torch.as_tensor(_DevArray(ptr.value, (num_q_heads, n_req, head_dim), "<i2"), device=dev)
        ob = num_q_heads * n_req * head_dim * 2
        lse = torch.as_tensor(_DevArray(ptr.value + ((ob + 255) & ~255), (num_q_heads, n_req), "<f4"), device=dev)
        return o.view(torch.bfloat16), lse

    def views_all(self, n_req: int, num_q_heads: int, head_dim: int, device=None):
        """(O [n_bufs][Hq][N][d] bf16, LSE [n_bufs][Hq][N] fp32): every buffer at once, strided."""
        import torch  # noqa: WPS433

        ptr = c_void_p()
        _check(lib().spa_peer_buffer(self.h, 0, ctypes.byref(ptr)))
        stride = (self.buf_bytes + 255) & ~255
        dev = device or torch.device("cuda", torch.cuda.current_device())
        H, N, d = num_q_heads, n_req, head_dim
        oa = _DevArray(ptr.value, (self.n_bufs, H, N, d), "<i2")
        oa.__cuda_array_interface__["strides"] = (stride, N * d * 2, d * 2, 2)
        ob = H * N * d * 2
        la = _DevArray(ptr.value + ((ob + 255) & ~255), (self.n_bufs, H, N), "<f4")
        la.__cuda_array_interface__["strides"] = (stride, N * 4, 4)
        return torch.as_tensor(oa, device=dev).view(torch.bfloat16), torch.as_tensor(la, device=dev)

    def status(self) -> int:
        st = c_int32()
        _check(lib().spa_peer_status(self.h, ctypes.byref(st)))
        return st.value

    def decode(self, plan: "Plan", layer: int, q_local, buf_idx: int, scale=None, with_lse=True, stream=None):
        d = q_local.shape[-1]
        if scale is None:
            scale = d ** -0.5
        if q_local.stride(2) != 1:
            raise ValueError("head_dim must be contiguous")
        _check(lib().spa_decode_attention_fused_gather(
            plan.h, self.h, int(layer), _ptr(q_local), q_local.stride(0), q_local.stride(1), int(buf_idx),
            int(bool(with_lse)), float(scale), _stream_ptr(stream)))

    def close(self):
        if self.h:
            _check(lib().spa_peer_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass
