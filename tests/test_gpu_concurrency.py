"""GPU: the boundary's threading contract.  The reference's transforms are
pure and safe to call concurrently; the C ABI promises the
same for a shared plan (include/fht_b200.h, fht_plan_create).  Host threads
hammer (a) the cached-plan int64 entry point fht2d_counted (transform.cpp:62-85)
and (b) one shared u8 batch Plan with staging and the concurrent K1 on the
plan's auxiliary stream, each thread on its own stream.  Every output must be
bit-exact against the oracle.
"""
import threading

import numpy as np
import pytest

import oracle
from paper_2411_07351_b200 import fht, workloads

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


def _run_threads(n, fn):
    errors = []

    def wrap(k):
        try:
            fn(k)
        except BaseException as e:  # noqa: BLE001 - reported below
            errors.append((k, repr(e)))

    ts = [threading.Thread(target=wrap, args=(k,)) for k in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors[:3]


def test_fht2d_counted_from_8_threads():
    """8 threads x 50 calls of fht2d_counted on 509x509 int64 images (int32
    accumulation on the device: K1P + the K1 tail block on the aux stream),
    one plan shared through the per-device cache."""
    rng = np.random.default_rng(123)
    imgs = [rng.integers(-1000, 1000, (509, 509)).astype(np.int64) for _ in range(6)]
    refs = [oracle.fht2d_counted_i64(im, oracle.TWEAKED) for im in imgs]
    bad = []

    def work(k):
        for it in range(50):
            i = (k + it) % len(imgs)
            ct = fht.fht2d_counted(imgs[i], "tweaked")
            if not np.array_equal(ct.hough, refs[i][0]) or ct.additions != refs[i][1]:
                bad.append((k, it, i))

    _run_threads(8, work)
    assert not bad, bad[:5]


def test_shared_u8_batch_plan_two_streams():
    """2 threads share one u8 batch plan (u16 pair mode, staging on, K1 forked
    onto the plan's aux stream), each on its own stream with its own inputs,
    outputs and workspace, 20 executes each with fresh inputs."""
    n_img, n = 8, 509
    plan = fht.Plan(n, n, "tweaked", in_dtype="u8", acc_dtype="i32", batch=n_img)
    assert plan.describe()["launches"] >= 4  # staging, K1P, K1, K2
    rng = np.random.default_rng(5)
    batches = [rng.integers(0, 256, (n_img, n, n), dtype=np.uint8) for _ in range(4)]
    # the oracle of every image of every batch (int32 tree, quadrant order)
    refs = []
    for b in batches:
        refs.append([oracle.fht2d_quadrants(b[i], oracle.TWEAKED, dtype=np.int32)[0] for i in range(n_img)])
    bad = []

    def work(k):
        st = torch.cuda.Stream()
        outs = plan.alloc_outputs()
        with torch.cuda.stream(st):
            xs = [torch.from_numpy(b).cuda() for b in batches]
            for it in range(20):
                j = (2 * it + k) % len(batches)
                plan(xs[j], out=outs, stream=st)
                st.synchronize()
                for i in (0, n_img // 2, n_img - 1):
                    for q in fht.QUADRANTS:
                        if not np.array_equal(outs[q][i].cpu().numpy(), refs[j][i][q]):
                            bad.append((k, it, i, q))

    _run_threads(2, work)
    assert not bad, bad[:5]


def test_plan_cache_is_bounded(monkeypatch):
    """The int64 entry points' plan cache keeps at most FHT_PLAN_CACHE plans
    (least recently used out) and can be cleared."""
    from paper_2411_07351_b200 import _lib

    lib = _lib.lib()
    lib.fht_plan_cache_clear(None)
    rng = np.random.default_rng(3)
    for w in range(20, 32):  # 12 sizes > the default cap of 8
        img = rng.integers(0, 50, (17, w))
        ct = fht.fht2d_counted(img)
        assert np.array_equal(ct.hough, oracle.fht2d_counted_i64(img)[0])
        assert lib.fht_plan_cache_size() <= 8
    import ctypes

    n = ctypes.c_size_t()
    assert lib.fht_plan_cache_clear(ctypes.byref(n)) == 0 and n.value == 8
    assert lib.fht_plan_cache_size() == 0
    # still works after a clear
    img = workloads.make_images("c1", 1)[0][:40, :40].astype(np.int64)
    assert np.array_equal(fht.fht2d(img), oracle.fht2d_counted_i64(img)[0])


def test_execute_makes_no_host_sync_or_allocation():
    """fht_execute is stream ordered: no stream synchronisation and no device
    allocation per call (debug counters of the library, torch's allocator)."""
    from paper_2411_07351_b200 import _lib

    imgs = workloads.make_images("c4", 8)
    plan = fht.Plan(509, 509, "tweaked", in_dtype="u8", acc_dtype="i32", batch=8)
    x = torch.from_numpy(imgs).cuda()
    out = plan.alloc_outputs()
    plan(x, out=out)
    torch.cuda.synchronize()
    c0, a0 = _lib.debug_counters(), torch.cuda.memory_stats()["allocation.all.allocated"]
    for _ in range(5):
        plan(x, out=out)
    assert _lib.debug_counters() == c0
    assert torch.cuda.memory_stats()["allocation.all.allocated"] == a0
    torch.cuda.synchronize()
    ref, _ = oracle.fht2d_quadrants(imgs[3], oracle.TWEAKED, dtype=np.int32)
    for q in fht.QUADRANTS:
        assert np.array_equal(out[q][3].cpu().numpy(), ref[q])
