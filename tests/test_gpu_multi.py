"""GPU tests of the multi-GPU path on one B200.

* shards with global offsets == one run (bitwise);
* survivor rebalancing inside dycl_run through the in-process transport (dycl_set_comm_local:
  world 2 / 3 graphs on this GPU, one host thread each -- the same plan, exchange, metadata and
  return code as the NCCL transport): rebalance on == off, bitwise, with rows actually moved,
  including a rank with an empty shard and a skewed split;
* the same with the exchange device-initiated (dycl_set_rebalance_mode DEVICE, SURVEY 8(f)1:
  counts, plan, row stores and results through the ranks' device windows, no host sync), over
  repeated runs (epochs / parity slots);
* the NCCL transport over torch's own communicator (world 1: the all-gather runs, no rows move),
  host and device modes (the latter registers an NCCL symmetric window and reads its LSA pointer);
* the min_margin output against the oracle's predicates.
"""
import os
import threading

import numpy as np
import pytest
import torch

import oracle as O
import workloads as wl
from oracle import programs as prg

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2307_04963_b200 import dycl as D  # noqa: E402
from paper_2307_04963_b200 import programs as P  # noqa: E402

DEV = torch.device("cuda:0")


def _run(model, x, g0=0, margin=False):
    B = x.shape[0]
    lg = torch.full((max(B, 1), model.K), float("nan"), device=DEV)
    pa = torch.full((max(B, 1),), -7, dtype=torch.int32, device=DEV)
    mm = torch.full((max(B, 1),), float("nan"), device=DEV) if margin else None
    model.run(x, lg, pa, global_offset=g0, min_margin=mm)
    torch.cuda.synchronize()
    out = (lg[:B].cpu().numpy(), pa[:B].cpu().numpy())
    return out + ((mm[:B].cpu().numpy(),) if margin else ())


@pytest.fixture(scope="module")
def r56w():
    return wl.sdn_r56_weights()


def test_shards_with_offsets_equal_one_run(r56w):
    X = torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, 0, 600)).to(DEV)
    m = P.build_sdn_resnet56(r56w, 600)
    l1, p1 = _run(m, X)
    la, pa = _run(m, X[:250].contiguous(), 0)
    lb, pb = _run(m, X[250:].contiguous(), 250)
    assert np.array_equal(np.concatenate([la, lb]), l1) and np.array_equal(np.concatenate([pa, pb]), p1)


def _rebalanced(builder, W, shards, policy=D.DYCL_REBALANCE_ALL, max_batch=None, mode=D.DYCL_REBALANCE_MODE_HOST,
                runs=1):
    """Run len(shards) graphs as ranks of one in-process group, one host thread each (device
    mode: the ranks' exchange kernels wait for one another through their windows, so every
    rank's run is in flight at once -- one stream per rank)."""
    world = len(shards)
    mb = max_batch or max(1, max(s.shape[0] for s in shards))
    models = [builder(W, mb) for _ in range(world)]
    grp = D.dycl_local_group_create(world)
    for r, m in enumerate(models):
        D.dycl_set_comm_local(m.g, grp, r, policy)
        D.dycl_set_rebalance_mode(m.g, mode)
    outs = [None] * world
    errs = []
    g0 = np.cumsum([0] + [s.shape[0] for s in shards])

    def work(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                B = shards[r].shape[0]
                lg = torch.full((max(B, 1), models[r].K), float("nan"), device=DEV)
                pa = torch.full((max(B, 1),), -7, dtype=torch.int32, device=DEV)
                mm = torch.full((max(B, 1),), float("nan"), device=DEV)
                for _ in range(runs):                 # repeated runs: epochs / parity slots advance
                    models[r].run(shards[r], lg, pa, stream=st, global_offset=int(g0[r]), min_margin=mm)
                st.synchronize()
                outs[r] = (lg[:B].cpu().numpy(), pa[:B].cpu().numpy(), mm[:B].cpu().numpy(),
                           D.dycl_rebalance_stats(models[r].g))
        except Exception as e:  # noqa: BLE001
            errs.append((r, e))

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    D.dycl_local_group_destroy(grp)
    return outs


def _skewed(X, paths, first_exit_share):
    """Order samples so rank 0 holds mostly the early-exiting ones (imbalance after exit 0)."""
    order = np.argsort(paths, kind="stable")
    return X[torch.from_numpy(order).to(DEV)], order


MODES = [D.DYCL_REBALANCE_MODE_HOST, D.DYCL_REBALANCE_MODE_DEVICE]


@pytest.mark.parametrize("mode", MODES, ids=["host", "device"])
@pytest.mark.parametrize("world,split", [(2, "equal"), (2, "skewed"), (3, "one_empty")])
def test_cfg2_rebalance_on_equals_off(r56w, world, split, mode):
    n = 900
    X = torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, 5000, n)).to(DEV)
    ref = P.build_sdn_resnet56(r56w, n)
    l_ref, p_ref, m_ref = _run(ref, X, margin=True)
    if split == "skewed":
        X, order = _skewed(X, p_ref, 0.5)
        l_ref, p_ref, m_ref = l_ref[order], p_ref[order], m_ref[order]
    if split == "one_empty":
        cuts = [0, 500, 500, n]
    else:
        cuts = [n * r // world for r in range(world + 1)]
    shards = [X[cuts[r]:cuts[r + 1]].contiguous() for r in range(world)]
    outs = _rebalanced(P.build_sdn_resnet56, r56w, shards, max_batch=max(c1 - c0 for c0, c1 in zip(cuts, cuts[1:])),
                       mode=mode, runs=3 if mode == D.DYCL_REBALANCE_MODE_DEVICE else 1)
    lg = np.concatenate([o[0] for o in outs])
    pg = np.concatenate([o[1] for o in outs])
    mg = np.concatenate([o[2] for o in outs])
    moved = sum(o[3][0] for o in outs)
    print(world, split, "rows moved", moved, [o[3] for o in outs])
    assert sum(o[3][0] for o in outs) == sum(o[3][1] for o in outs)
    if split != "equal":
        assert moved > 0
    assert np.array_equal(pg, p_ref)
    assert np.array_equal(lg, l_ref)
    assert np.array_equal(mg, m_ref)


@pytest.mark.parametrize("mode", MODES, ids=["host", "device"])
def test_cfg5_rebalance_on_equals_off(mode):
    W = wl.resnet50_ee_weights()
    n = 96
    X = wl.image_inputs_torch(wl.INPUT_SEED, 900, n, hw=224, device="cuda")
    ref = P.build_resnet50_ee(W, n)
    l_ref, p_ref = _run(ref, X)
    X, order = _skewed(X, p_ref, 0.5)
    l_ref, p_ref = l_ref[order], p_ref[order]
    shards = [X[:n // 2].contiguous(), X[n // 2:].contiguous()]
    outs = _rebalanced(P.build_resnet50_ee, W, shards, max_batch=n // 2, mode=mode)
    moved = sum(o[3][0] for o in outs)
    print("cfg5 rows moved", moved)
    assert moved > 0
    assert np.array_equal(np.concatenate([o[1] for o in outs]), p_ref)
    assert np.array_equal(np.concatenate([o[0] for o in outs]), l_ref)


@pytest.mark.parametrize("mode", MODES, ids=["host", "device"])
def test_rebalance_policy_first_exit_only(r56w, mode):
    n = 400
    X = torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, 7000, n)).to(DEV)
    l_ref, p_ref = _run(P.build_sdn_resnet56(r56w, n), X)
    X, order = _skewed(X, p_ref, 0.5)
    outs = _rebalanced(P.build_sdn_resnet56, r56w, [X[:200].contiguous(), X[200:].contiguous()], policy=1,
                       max_batch=200, mode=mode)
    assert np.array_equal(np.concatenate([o[1] for o in outs]), p_ref[order])
    assert np.array_equal(np.concatenate([o[0] for o in outs]), l_ref[order])


@pytest.mark.parametrize("mode", MODES, ids=["host", "device"])
def test_nccl_transport_world1(r56w, mode):
    """dycl_set_comm with torch's own NCCL communicator (world 1: the count all-gather runs on
    NCCL every exit, no rows move); results equal the plain run."""
    import torch.distributed as dist
    from paper_2307_04963_b200 import dist as DI
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29531")
    created = False
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
        created = True
    try:
        n = 256
        X = torch.from_numpy(wl.image_inputs(wl.INPUT_SEED, 11000, n)).to(DEV)
        l_ref, p_ref = _run(P.build_sdn_resnet56(r56w, n), X)
        m = P.build_sdn_resnet56(r56w, n)
        D.dycl_set_comm(m.g, DI.nccl_comm_ptr(), 0, 1, D.DYCL_REBALANCE_ALL)
        D.dycl_set_rebalance_mode(m.g, mode)
        l1, p1 = _run(m, X)
        l1, p1 = _run(m, X)
        assert np.array_equal(p1, p_ref) and np.array_equal(l1, l_ref)
        assert D.dycl_rebalance_stats(m.g) == (0, 0)
    finally:
        if created:
            dist.destroy_process_group()


def test_min_margin_matches_oracle_predicates(r56w):
    """min_margin = min over the predicates along the sample's path of |p - tau| (R12): the
    GPU's value vs the oracle's (mirror) predicates."""
    n = 128
    Xn = wl.image_inputs(wl.INPUT_SEED, 3000, n)
    m = P.build_sdn_resnet56(r56w, n)
    lg, pg, mg = _run(m, torch.from_numpy(Xn).to(DEV), margin=True)
    _, po, pr = O.run_batch(O.sdn_resnet56, Xn, prg.prepare(r56w), "mirror")
    ora = np.array([min([abs(v - t) for (_, v, t) in p], default=np.inf) for p in pr])
    same = pg == po
    assert same.sum() >= n - 2
    assert np.all(np.abs(mg[same] - ora[same]) <= 5e-3), np.max(np.abs(mg[same] - ora[same]))
    assert np.all(mg >= 0)
