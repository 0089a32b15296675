"""Image-parallel rendering over R shards on the GPU.

The R-way split (Gaussians by contiguous id range, the view by column strips, records and 9-float
screen-space gradients exchanged) must reproduce the unsplit render:
  * strip images assembled side by side == the single-GPU image == the reference oracle, bit for bit
    (per-pixel contribution lists and their order are unchanged);
  * the loss (fp64 strip sums added in strip order, cast once) == the unsplit loss;
  * gradients within the north-star fp32 tolerance rel_err <= 1e-4 (straddling Gaussians add their
    strips' partials in strip order: the reference's split aggregation, splitter.hpp:85-123).
The two-process test runs the real torch.distributed path (gloo, host-staged: both ranks share this
one GPU) and must equal the in-process simulation bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracles as O
import paper_2509_15645_b200 as G
from paper_2509_15645_b200 import dist as D
from paper_2509_15645_b200 import imgpar as IP

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def scene(seed, n, w, h):
    cfg = G.SynthConfig(seed=seed, n=n, cams=4, width=w, height=h)
    rows, cams = G.synth_scene_params(cfg)
    gts = [G.render_view(torch.from_numpy(rows).cuda(), c, 3) for c in cams]
    start = rows.copy()
    start[:, 10] = np.float32(np.log(0.1 / 0.9))
    start[:, 14:] = 0.0
    return start, cams, gts


def shard_scenes(rows_t, cam, vp, R):
    n = rows_t.shape[0]
    geo = rows_t[:, :10].contiguous()
    ng = rows_t[:, 10:].contiguous()
    out = []
    for r in range(R):
        lo, hi = D.id_range(n, r, R)
        g, q = geo[lo:hi].contiguous(), ng[lo:hi].contiguous()
        ids = G.frustum_cull(g, hi - lo, cam, vp)
        out.append((lo, G.RenderScene(ids=ids, geo=g, nongeo=q)))
    return out


def unsplit(rows_t, cam, vp, gt):
    geo = rows_t[:, :10].contiguous()
    ng = rows_t[:, 10:].contiguous()
    ids = G.frustum_cull(geo, geo.shape[0], cam, vp)
    sc = G.RenderScene(ids=ids, geo=geo, nongeo=ng)
    fw = G.rasterize_forward(sc, cam, vp, gt=gt)
    gb = G.rasterize_backward(sc, cam, fw, fw.d_img)
    return ids, fw, gb


@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("seed,n,w,h", [(3, 3000, 96, 64), (17, 20000, 200, 120)])
def test_simulated_split_equals_unsplit(seed, n, w, h, R):
    rows, cams, gts = scene(seed, n, w, h)
    rows_t = torch.from_numpy(rows).cuda()
    vp = G.viewport_full(w, h)
    for ci in range(2):
        cam, gt = cams[ci], gts[ci]
        ids, fw, gb = unsplit(rows_t, cam, vp, gt)
        shards = shard_scenes(rows_t, cam, vp, R)
        loss, grads, image = IP.simulate_render([s for _, s in shards], cam, vp, gt)
        torch.cuda.synchronize()
        # global id list = shard lists + offsets, in shard order
        glob = torch.cat([s.ids.long() + lo for lo, s in shards]).cpu().numpy()
        assert np.array_equal(glob, ids.cpu().numpy())
        assert np.array_equal(bits(image.cpu().numpy()), bits(fw.image.cpu().numpy()))
        assert loss == float(fw.loss.item())
        rows_split = torch.cat([g.rows for g in grads]).cpu().numpy()
        m2d_split = torch.cat([g.mean2d for g in grads]).cpu().numpy()
        rel = float(O.rel_err(rows_split, gb.rows.cpu().numpy()).max(initial=0.0))
        relm = float(O.rel_err(m2d_split, gb.mean2d.cpu().numpy()).max(initial=0.0))
        assert rel <= 1e-4 and relm <= 1e-4, (rel, relm)
        if R == 1:  # one strip: the same sums in the same order (up to 0 + x)
            assert np.array_equal(rows_split, gb.rows.cpu().numpy())


def test_split_image_equals_oracle(orc):
    rows, cams, gts = scene(5, 2000, 64, 48)
    cam = cams[1]
    vp = G.viewport_full(64, 48)
    rows_t = torch.from_numpy(rows).cuda()
    shards = shard_scenes(rows_t, cam, vp, 3)
    loss, grads, image = IP.simulate_render([s for _, s in shards], cam, vp, gts[1])
    geo, ng = rows[:, :10].copy(), rows[:, 10:].copy()
    cam_arr = O.cam_from_struct(cam)
    want_ids = O.orc_cull(geo, cam_arr, [0, 64, 0, 48])
    ref = O.render("orc", want_ids, geo, ng, cam_arr, [0, 64, 0, 48], gt=gts[1].cpu().numpy())
    assert np.array_equal(bits(image.cpu().numpy()), bits(ref["image"]))
    assert loss == ref["loss"]
    rows_split = torch.cat([g.rows for g in grads]).cpu().numpy()
    assert float(O.rel_err(rows_split, ref["rows"]).max(initial=0.0)) <= 1e-4


def test_routing_sets_and_order():
    rows, cams, _ = scene(9, 5000, 160, 96)
    rows_t = torch.from_numpy(rows).cuda()
    cam = cams[0]
    vp = G.viewport_full(160, 96)
    geo = rows_t[:, :10].contiguous()
    ids = G.frustum_cull(geo, geo.shape[0], cam, vp)
    sc = G.RenderScene(ids=ids, geo=geo, nongeo=rows_t[:, 10:].contiguous())
    recs = G.project(sc, cam, vp)
    box = recs.view(torch.int32)[:, 12:16].cpu().numpy()  # bx0, bx1, by0, by1
    bounds = IP.strip_bounds(0, 160, 4)
    slots, counts = G.route_strips(recs, bounds)
    for k in range(4):
        want = np.nonzero((box[:, 1] > box[:, 0]) & (box[:, 3] > box[:, 2]) & (box[:, 0] < bounds[k + 1]) &
                          (box[:, 1] > bounds[k]))[0]
        got = slots[k, : counts[k]].cpu().numpy()
        assert np.array_equal(got, want)  # ascending slots, exactly the touching set


def test_empty_strips_and_empty_shards():
    # more strips than 16-px tile columns: some strips are empty windows; a shard may see nothing
    rows, cams, gts = scene(21, 300, 48, 40)
    rows_t = torch.from_numpy(rows).cuda()
    vp = G.viewport_full(48, 40)
    cam, gt = cams[0], gts[0]
    ids, fw, gb = unsplit(rows_t, cam, vp, gt)
    shards = shard_scenes(rows_t, cam, vp, 8)
    loss, grads, image = IP.simulate_render([s for _, s in shards], cam, vp, gt)
    assert np.array_equal(bits(image.cpu().numpy()), bits(fw.image.cpu().numpy()))
    assert loss == float(fw.loss.item())
    rows_split = torch.cat([g.rows for g in grads]).cpu().numpy()
    assert float(O.rel_err(rows_split, gb.rows.cpu().numpy()).max(initial=0.0)) <= 1e-4


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        rows, cams, gts = scene(3, 3000, 96, 64)
        rows_t = torch.from_numpy(rows).cuda()
        vp = G.viewport_full(96, 64)
        cam = cams[1]
        lo, sc = shard_scenes(rows_t, cam, vp, world)[rank]
        ex = IP.TorchExchange()
        loss, gb, image, info = IP.render_step(ex, sc, cam, vp, gts[1])
        torch.cuda.synchronize()
        q.put((rank, loss, gb.rows.cpu().numpy(), image.cpu().numpy(), info["bounds"]))
    finally:
        dist.destroy_process_group()


def test_two_process_render_step_equals_simulation():
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rows, cams, gts = scene(3, 3000, 96, 64)
    rows_t = torch.from_numpy(rows).cuda()
    vp = G.viewport_full(96, 64)
    shards = shard_scenes(rows_t, cams[1], vp, world)
    loss, grads, image = IP.simulate_render([s for _, s in shards], cams[1], vp, gts[1])
    assert res[0][1] == res[1][1] == loss
    for r in range(world):
        assert np.array_equal(bits(res[r][2]), bits(grads[r].rows.cpu().numpy()))
    full = np.concatenate([res[0][3], res[1][3]], axis=1)
    assert np.array_equal(bits(full), bits(image.cpu().numpy()))


@pytest.mark.parametrize("pipelined", [False, True])
def test_shard_trainer_world1_equals_engine(pipelined):
    rows, cams, gts = scene(13, 4000, 80, 64)
    tr = IP.ShardTrainer(rows, cams, gts, pipelined=pipelined)
    losses = [tr.step() for _ in range(6)]
    tr.drain()
    torch.cuda.synchronize()
    eng = G.OffloadEngine(rows, cams, np.stack([g.cpu().numpy() for g in gts]), pipelined=False)
    el, _ = eng.run(6)
    st = eng.state()
    eng.close()
    assert np.array_equal(np.float32(losses), el)
    for k in ("geo_w", "ng_w", "ng_m", "ng_v"):
        assert np.array_equal(tr.state()[k].cpu().numpy(), st[k]), k  # == (signed zeros compare equal)
    assert np.array_equal(tr.state()["ng_counter"].cpu().numpy(), st["ng_counter"])


def test_shard_trainer_densify_stats_and_device_loss_equal_engine():
    """The shard keeps the engine's densification statistics (engine.hpp:404-408) bit for bit, and
    device_loss=True returns the same loss as a device scalar (no per-step host round trip)."""
    rows, cams, gts = scene(13, 4000, 80, 64)
    tr = IP.ShardTrainer(rows, cams, gts, device_loss=True, balance=True)
    losses = [tr.step() for _ in range(6)]
    assert all(isinstance(x, torch.Tensor) and x.is_cuda for x in losses)
    tr.drain()
    torch.cuda.synchronize()
    eng = G.OffloadEngine(rows, cams, np.stack([g.cpu().numpy() for g in gts]), pipelined=False)
    el, _ = eng.run(6)
    norm, cnt = eng.accum()
    eng.close()
    assert np.array_equal(np.float32([float(x) for x in losses]), el)
    assert np.array_equal(tr.accum_cnt.cpu().numpy(), cnt)
    assert np.array_equal(tr.accum_norm.cpu().numpy().view(np.uint64), np.asarray(norm).view(np.uint64))


def _train_worker(rank, world, port, q, balance=False):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        rows, cams, gts = scene(13, 4000, 80, 64)
        lo, hi = D.id_range(rows.shape[0], rank, world)
        tr = IP.ShardTrainer(rows[lo:hi], cams, gts, IP.TorchExchange(), balance=balance)
        losses = [tr.step() for _ in range(5)]
        tr.drain()
        torch.cuda.synchronize()
        q.put((rank, losses, tr.state()["geo_w"].cpu().numpy(), tr.state()["ng_w"].cpu().numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("balance", [False, True])
def test_two_process_training_matches_single_shard(balance):
    """Two shards over gloo (equal strips, or strips balanced by visible Gaussians) train like one."""
    import torch.multiprocessing as mp

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_train_worker, args=(r, world, port, q, balance)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rows, cams, gts = scene(13, 4000, 80, 64)
    tr = IP.ShardTrainer(rows, cams, gts)
    losses = [tr.step() for _ in range(5)]
    tr.drain()
    # the forward of iteration 0 sees identical parameters: bit-identical loss
    assert res[0][1][0] == res[1][1][0] == losses[0]
    assert np.allclose(res[0][1], losses, rtol=1e-4, atol=0)
    geo = np.concatenate([res[0][2], res[1][2]])
    ng = np.concatenate([res[0][3], res[1][3]])
    assert float(O.rel_err(geo, tr.state()["geo_w"].cpu().numpy()).max()) <= 1e-4
    assert float(O.rel_err(ng, tr.state()["ng_w"].cpu().numpy()).max()) <= 1e-4
