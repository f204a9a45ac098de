"""ctypes binding of ``libslbm_b200.so`` (declarations: include/slbm_b200.h).

There is no fallback: if the library is missing or cannot load, every
engine constructor raises.  The library is built in-tree by
``paper_2408_06880_b200.build`` / ``__graft_entry__.build()``.
"""

from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libslbm_b200.so")

c_i64p = C.POINTER(C.c_int64)
c_i32p = C.POINTER(C.c_int32)
c_u8p = C.POINTER(C.c_uint8)
c_u32p = C.POINTER(C.c_uint32)
c_dp = C.POINTER(C.c_double)
vp = C.c_void_p


class SlbmInfo(C.Structure):
    _fields_ = [
        ("q", C.c_int32),
        ("dim", C.c_int32),
        ("pattern", C.c_int32),
        ("parity", C.c_int32),
        ("has_split", C.c_int32),
        ("model", C.c_int32),
        ("n_fluid", C.c_int64),
        ("total_slots", C.c_int64),
        ("n_ubb_slots", C.c_int64),
        ("n_ghost_slots", C.c_int64),
        ("n_interior", C.c_int64),
        ("n_frame", C.c_int64),
        ("base", C.c_int64 * 28),
        ("n_ubb_q", C.c_int64 * 27),
        ("n_ghost_q", C.c_int64 * 27),
        ("device_bytes", C.c_int64),
        ("n_outlet_slots", C.c_int64),
        ("layout", C.c_int64),
    ]


# name -> argtypes (restype is int for every function except the two string getters)
SIGNATURES = {
    "slbm_engine_create": [c_u8p, c_dp, C.c_int, c_i32p, c_u8p, C.c_int, C.c_int, C.c_double,
                           C.c_double, C.c_int, c_i32p, C.c_int, C.POINTER(vp)],
    "slbm_engine_create_dense": [c_u8p, c_dp, C.c_int, c_i32p, c_u8p, C.c_int, C.c_int,
                                 C.c_double, C.c_double, C.c_int, c_i32p, C.c_int, C.POINTER(vp)],
    "slbm_engine_destroy": [vp],
    "slbm_engine_info": [vp, C.POINTER(SlbmInfo)],
    "slbm_engine_stream": [vp, C.POINTER(vp)],
    "slbm_engine_set_stream": [vp, vp],
    "slbm_engine_set_params": [vp, C.c_int, C.c_double, C.c_double],
    "slbm_engine_set_cumulant_rates": [vp, C.c_double, C.POINTER(C.c_double), C.c_int],
    "slbm_export_lists": [vp, c_u32p, c_i64p, c_i64p, c_i64p, c_dp, c_i64p, c_i64p, c_i64p],
    "slbm_export_split": [vp, c_i64p, c_i64p],
    "slbm_init_canonical": [vp, c_dp],
    "slbm_init_canonical_dev": [vp, vp],
    "slbm_init_equilibrium": [vp, c_dp, C.c_int, c_dp, C.c_int],
    "slbm_canonical_state": [vp, c_dp],
    "slbm_macroscopic": [vp, c_dp, c_dp],
    "slbm_macroscopic_compact": [vp, C.POINTER(C.c_double), C.POINTER(C.c_double)],
    "slbm_total_mass": [vp, c_dp],
    "slbm_total_moments": [vp, c_dp],
    "slbm_macroscopic_global": [vp, vp, vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "slbm_copy_to_host": [vp, vp, C.c_int64, C.c_int],
    "slbm_engine_sweep_ctas": [vp, C.POINTER(C.c_int)],
    "slbm_refresh_boundary": [vp, C.c_int],
    "slbm_step": [vp, C.c_int],
    "slbm_finish_step": [vp],
    "slbm_run": [vp, C.c_int64, C.c_int],
    "slbm_poll_instability": [vp, c_i64p],
    "slbm_synchronize": [vp],
    "slbm_parity": [vp, C.POINTER(C.c_int)],
    "slbm_set_parity": [vp, C.c_int],
    "slbm_buffer_state": [vp, C.POINTER(C.c_int)],
    "slbm_slot_index": [vp, c_i64p, c_i64p, C.c_int64, c_i64p],
    "slbm_ghost_slot_index": [vp, c_i64p, c_i64p, C.c_int64, c_i64p],
    "slbm_read_slots": [vp, c_i64p, C.c_int64, c_dp],
    "slbm_write_slots": [vp, c_i64p, C.c_int64, c_dp],
    "slbm_pdf_pointer": [vp, C.POINTER(vp)],
    "slbm_export_cid_map": [vp, C.POINTER(C.c_int32)],
    "slbm_poll_engines": [C.POINTER(vp), C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int)],
    "slbm_pdf_layout": [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "slbm_halo_create": [C.c_int, C.POINTER(vp)],
    "slbm_halo_destroy": [vp],
    "slbm_halo_add_local": [vp, C.c_int, vp, vp, c_i64p, C.c_int64, c_i64p, c_i64p, C.c_int64],
    "slbm_halo_add_send": [vp, C.c_int, vp, C.c_int, c_i64p, C.c_int64],
    "slbm_halo_add_recv": [vp, C.c_int, vp, C.c_int, C.c_int64, c_i64p, c_i64p, C.c_int64],
    "slbm_halo_commit": [vp, vp],
    "slbm_halo_start": [vp, C.c_int, vp],
    "slbm_halo_wait": [vp, vp],
    "slbm_halo_peer_sizes": [vp, C.c_int, C.c_int, c_i64p, c_i64p],
    "slbm_halo_pack_host": [vp, C.c_int, C.c_int, c_dp],
    "slbm_halo_unpack_host": [vp, C.c_int, C.c_int, c_dp],
    "slbm_halo_local": [vp, C.c_int],
    "slbm_halo_start_ex": [vp, C.c_int, vp, C.c_int],
    "slbm_halo_local_on": [vp, C.c_int, vp],
    "slbm_engine_set_frame": [vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)],
    "slbm_nccl_comm_init": [vp, C.c_int, C.c_int, C.c_int, C.POINTER(vp)],
    "slbm_nccl_get_unique_id": [vp],
    "slbm_nccl_comm_destroy": [vp],
    "slbm_halo_use_peer": [vp, C.c_int],
    "slbm_halo_ipc_handles": [vp, vp, vp],
    "slbm_halo_recv_section": [vp, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "slbm_halo_connect": [vp, C.c_int, vp, vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "slbm_voxelize_spheres": [c_i32p, c_dp, C.c_int64, C.c_double, C.c_int, c_u8p],
    "slbm_set_tuning": [C.c_int, C.c_int],
    "slbm_engine_set_tuning": [vp, C.c_int, C.c_int],
    "slbm_launch_count": [C.POINTER(C.c_int64)],
    "slbm_group_create": [C.POINTER(vp), C.c_int, C.POINTER(vp)],
    "slbm_group_destroy": [vp],
    "slbm_group_refresh": [vp, C.c_int, vp],
    "slbm_group_boundary": [vp, vp, C.c_int, C.c_int, vp],
    "slbm_group_step": [vp, C.c_int, vp],
    "slbm_group_finish": [vp, vp],
    "slbm_group_link_halo": [vp, vp],
    "slbm_group_stale_copy": [vp, C.c_int, vp],
    "slbm_capture_begin": [vp],
    "slbm_capture_end": [vp, C.POINTER(vp)],
    "slbm_graph_launch": [vp, vp],
    "slbm_graph_destroy": [vp],
    "slbm_last_error": [],
    "slbm_version": [],
}

_lib = None


def load() -> C.CDLL:
    """Load the library once; raise loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -m paper_2408_06880_b200.build); there is no CPU fallback"
        )
    lib = C.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_char_p if name in ("slbm_last_error", "slbm_version") else C.c_int
    _lib = lib
    return lib


def call(name: str, *args) -> None:
    lib = load()
    status = getattr(lib, name)(*args)
    if status != 0:
        msg = lib.slbm_last_error().decode(errors="replace")
        errors.raise_for_status(status, msg)


def ptr(arr, ctype):
    """Pointer into a contiguous numpy array (or None)."""
    if arr is None:
        return None
    return arr.ctypes.data_as(C.POINTER(ctype))


def launch_count() -> int:
    """Kernels of this library launched so far in the process
    (slbm_launch_count; graph replays included)."""
    n = C.c_int64(0)
    call("slbm_launch_count", C.byref(n))
    return int(n.value)
