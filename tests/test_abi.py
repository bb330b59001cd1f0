"""CPU-side checks of the C ABI: the library loads, exports every symbol
include/qlm.h declares, the ctypes/numpy struct mirrors match the C layout,
and host-side validation rejects bad inputs with a message naming the field
(validation runs before any CUDA call, so no GPU is touched)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2407_00047_b200 import _lib as L
from paper_2407_00047_b200 import build as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "qlm.h")


@pytest.fixture(scope="module")
def lib():
    B.build()
    return L.lib()


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"QLM_API\s+[\w\s\*]+?\b(qlm_\w+)\s*\(", src)))


def test_every_declared_symbol_is_exported(lib):
    names = declared()
    assert len(names) >= 15
    out = subprocess.check_output(["nm", "-D", "--defined-only", L.LIB_PATH], text=True)
    exported = set(re.findall(r" T (qlm_\w+)", out))
    assert set(names) <= exported, set(names) - exported
    assert set(names) == set(L.SIGNATURES), "ctypes signatures out of sync with qlm.h"
    for n in names:
        assert hasattr(lib, n)
    # nothing but the ABI is exported
    assert exported == set(names)


def test_library_is_sm100a_only():
    out = subprocess.check_output(["cuobjdump", "--list-elf", L.LIB_PATH], text=True)
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_struct_layout_matches_c(tmp_path):
    probe = tmp_path / "probe.c"
    probe.write_text(r'''
#include <stdio.h>
#include <stddef.h>
#include "qlm.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(qlm_group), sizeof(qlm_queue),
         sizeof(qlm_profile), sizeof(qlm_len_tables), sizeof(qlm_options), sizeof(qlm_record),
         sizeof(qlm_candidates), sizeof(qlm_best));
  printf("%zu %zu %zu %zu %zu %zu\n", offsetof(qlm_group, slo_s), offsetof(qlm_group, dist_id),
         offsetof(qlm_queue, backlog_mean_s), offsetof(qlm_candidates, first_from),
         offsetof(qlm_candidates, seed), offsetof(qlm_candidates, moves));
  printf("%zu %zu %zu %zu\n", sizeof(qlm_tiers), sizeof(qlm_requests), offsetof(qlm_requests, model),
         offsetof(qlm_requests, feat));
  return 0;
}''')
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(probe), "-o", str(exe)])
    a, b, c = subprocess.check_output([str(exe)], text=True).strip().split("\n")
    assert [int(x) for x in c.split()] == [C.sizeof(L.Tiers), C.sizeof(L.Requests), L.Requests.model.offset,
                                           L.Requests.feat.offset]
    sizes = [int(x) for x in a.split()]
    assert sizes == [L.GROUP_DTYPE.itemsize, L.QUEUE_DTYPE.itemsize, C.sizeof(L.Profile),
                     C.sizeof(L.LenTables), C.sizeof(L.Options), C.sizeof(L.Record),
                     C.sizeof(L.Candidates), C.sizeof(L.Best)]
    offs = [int(x) for x in b.split()]
    assert offs == [L.GROUP_DTYPE.fields["slo_s"][1], L.GROUP_DTYPE.fields["dist_id"][1],
                    L.QUEUE_DTYPE.fields["backlog_mean_s"][1], L.Candidates.first_from.offset,
                    L.Candidates.seed.offset, L.Candidates.moves.offset]


def _create(lib, groups, queues, D=1, M=1, theta=1000.0, swap_diag=0.0, K=None, opt=None):
    arrs = [np.full((D, M), theta), np.full((D, M), 0.5), np.full((D, M), 1.2),
            np.full((D, M), 0.025), np.full((D, M), 2048.0)]
    sw = np.zeros((D, M, M))
    sw[0, 0, 0] = swap_diag
    arrs.append(sw)
    prof = L.Profile(D, M, *[a.ctypes.data for a in arrs])
    tabs = None
    if K is not None:
        t = np.ones((1, max(K, 1)), np.uint16)
        tabs = L.LenTables(K, 1, t.ctypes.data)
    h = C.c_void_p()
    rc = lib.qlm_create(groups.ctypes.data if groups is not None else None,
                        0 if groups is None else len(groups), queues.ctypes.data, len(queues),
                        C.byref(prof), C.byref(tabs) if tabs else None,
                        C.byref(opt) if opt else None, C.byref(h))
    return rc, lib.qlm_last_error().decode()


def _good():
    g = np.zeros(3, L.GROUP_DTYPE)
    g["n_req"], g["slo_s"], g["mu_out"], g["var_out"], g["dist_id"] = 4, 20.0, 100.0, 50.0, -1
    q = np.zeros(2, L.QUEUE_DTYPE)
    return g, q


@pytest.mark.parametrize("field,value,needle", [
    ("model", 3, "groups[1].model=3"),
    ("n_req", 0, "groups[1].n_req=0"),
    ("slo_s", 0.0, "groups[1].slo_s"),
    ("slo_s", np.inf, "groups[1].slo_s"),
    ("mu_out", -1.0, "groups[1].mu_out"),
    ("var_out", np.nan, "groups[1].var_out"),
    ("dist_id", 0, "groups[1].dist_id=0"),
    ("reserved", 1, "groups[1].reserved"),
])
def test_group_validation_names_field(lib, field, value, needle):
    g, q = _good()
    g[field][1] = value
    rc, msg = _create(lib, g, q)
    assert rc == L.QLM_EINVAL and needle in msg


def test_queue_and_profile_validation(lib):
    g, q = _good()
    q["device"][1] = 2
    rc, msg = _create(lib, g, q)
    assert rc == L.QLM_EINVAL and "queues[1].device=2" in msg
    g, q = _good()
    q["resident_model"][0] = -1
    rc, msg = _create(lib, g, q)
    assert rc == L.QLM_EINVAL and "queues[0].resident_model" in msg
    g, q = _good()
    q["backlog_mean_s"][1] = -3.0
    rc, msg = _create(lib, g, q)
    assert rc == L.QLM_EINVAL and "backlog_mean_s" in msg
    g, q = _good()
    rc, msg = _create(lib, g, q, theta=0.0)
    assert rc == L.QLM_EINVAL and "theta[0][0]" in msg
    rc, msg = _create(lib, g, q, swap_diag=1.5)
    assert rc == L.QLM_EINVAL and "swap_s[0][0][0]" in msg and "diagonal" in msg
    rc, msg = _create(lib, None, q)
    assert rc == L.QLM_EINVAL and "G=0" in msg
    rc, msg = _create(lib, g, q, K=3)
    assert rc == L.QLM_EINVAL and "tabs.K=3" in msg
    rc, msg = _create(lib, g, q, opt=L.Options(-1.0, 0.01, 0, 0))
    assert rc == L.QLM_EINVAL and "z_clamp" in msg
    big = np.zeros(40000, L.GROUP_DTYPE)
    rc, msg = _create(lib, big, q)
    assert rc == L.QLM_ERANGE and "32768" in msg


def test_total_requests_below_2_pow_24(lib):
    # S1's clamped-slot numerator is an fp32 sum of n_i: exact below 2^24 (R11)
    g = np.zeros(2, L.GROUP_DTYPE)
    g["n_req"], g["slo_s"], g["mu_out"], g["dist_id"] = [1 << 23, (1 << 23) - 1], 10.0, 100.0, -1
    q = np.zeros(1, L.QUEUE_DTYPE)
    rc, msg = _create(lib, g, q)
    assert rc != L.QLM_ERANGE                          # 2^24 - 1 requests: accepted (no GPU -> ECUDA)
    g["n_req"][1] = 1 << 23
    rc, msg = _create(lib, g, q)
    assert rc == L.QLM_ERANGE and "2^24" in msg


def test_null_context_calls_fail_cleanly(lib):
    cand = L.Candidates(L.CAND_RANDOM, 1, None, 0, 1, 0, 10, None)
    assert lib.qlm_score_orderings(None, C.byref(cand), None, None, None, None) == L.QLM_EINVAL
    assert lib.qlm_rwt_estimate(None, C.byref(cand), None, None, None, None) == L.QLM_EINVAL
    assert lib.qlm_dims(None, None, None, None, None, None) == L.QLM_EINVAL
    assert lib.qlm_adopt_best(None, C.byref(cand), None, None, None) == L.QLM_EINVAL
    assert lib.qlm_local_search(None, None, 1, 2, 64, 1, 1, None, None) == L.QLM_EINVAL
    lib.qlm_destroy(None)
    assert lib.qlm_abi_version() == 4


def test_comm_calls_validate_on_the_host(lib):
    # the communicator entry points reject bad arguments before
    # touching CUDA or NCCL
    buf = (C.c_uint8 * L.COMM_ID_BYTES)()
    assert lib.qlm_comm_unique_id(None) == L.QLM_EINVAL
    assert lib.qlm_comm_attach(None, buf, 0, 1) == L.QLM_EINVAL
    assert lib.qlm_comm_detach(None) == L.QLM_EINVAL
    assert lib.qlm_comm_info(None, None, None, None) == L.QLM_EINVAL
    assert "NULL" in lib.qlm_last_error().decode()


def test_comm_unique_id_needs_no_gpu(lib):
    # NCCL is resolved at run time (dlopen); the unique id is host-side bootstrap
    # state, so it can be made on the CPU host; without NCCL the call names it
    buf = (C.c_uint8 * L.COMM_ID_BYTES)()
    rc = lib.qlm_comm_unique_id(buf)
    if rc == L.QLM_OK:
        assert any(bytes(buf))
    else:
        assert rc == L.QLM_ENCCL and "nccl" in lib.qlm_last_error().decode().lower()


def test_form_groups_host_validation(lib):
    # Alg. 1 entry point (R21): sizes are checked on the host before any CUDA call
    dummy = C.c_void_p(16)
    G, it = C.c_int32(), C.c_int32()

    def call(n=10, dims=2, M=2, k=(2, 2), limit=8, max_iter=5, lab=dummy, gof=dummy):
        r = L.Requests(n, dims, dummy, dummy, dummy, dummy)
        ka = np.asarray(k, np.int32)
        rc = lib.qlm_form_groups(C.byref(r), M, ka.ctypes.data, limit, max_iter, lab, gof, dummy, 4,
                                 C.byref(G), C.byref(it), 0, None)
        return rc, lib.qlm_last_error().decode()

    for kw, msg in [(dict(n=0), "req.n"), (dict(dims=5), "req.dims"), (dict(M=0, k=()), "M="),
                    (dict(k=(0, 2)), "k_per_model[0]"), (dict(k=(1000, 1000)), "sum of k_per_model"),
                    (dict(limit=0), "limit"), (dict(limit=40000), "limit"), (dict(max_iter=0), "max_iter"),
                    (dict(lab=None), "label_of")]:
        rc, err = call(**kw)
        assert rc == L.QLM_EINVAL and msg in err, (kw, rc, err)


def test_missing_library_fails_loudly(tmp_path):
    # no CPU fallback: with the extension absent, the binding raises on first use
    code = ("import paper_2407_00047_b200 as q\n"
            "try:\n    q._lib.lib()\nexcept RuntimeError as e:\n    print('RAISED', e)\n")
    env = dict(os.environ, QLM_LIB_PATH=str(tmp_path / "absent" / "libqlm.so"))
    out = subprocess.check_output([os.sys.executable, "-c", code], env=env, text=True, cwd=ROOT)
    assert out.startswith("RAISED") and "not built" in out


def test_qlm_create_without_gpu_is_a_named_error(lib):
    # on a host without an sm_100 device the library refuses instead of falling back
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2407_00047_b200 import RwtEstimator
    from workloads.synth import make_config
    with pytest.raises(L.QlmError, match="CUDA device|sm_"):
        RwtEstimator(make_config("C1"))


def test_kernel_override_flags_match_header(lib):
    # every QLM_OVERRIDE_* bit of qlm.h is named in the Python binding, ALL is
    # their union, and an unknown bit is a named error (host-only call)
    src = open(HEADER).read()
    bits = {m.group(1).lower(): int(m.group(2)) for m in
            re.finditer(r"#define QLM_OVERRIDE_(\w+) (\d+)u", src) if m.group(1) != "ALL"}
    assert bits == L.OVERRIDE
    every = int(re.search(r"#define QLM_OVERRIDE_ALL (\d+)u", src).group(1))
    assert every == sum(bits.values())
    assert lib.qlm_set_kernel_overrides(every + 1, 0) != 0
    assert lib.qlm_set_kernel_overrides(every, 0) == 0
    assert lib.qlm_set_kernel_overrides(0, 0) == 0
