"""salt-bench (GPU CSV sweep, reference bench.py contract) and the static
traffic counter — CPU parts; a small GPU sweep is gpu-marked."""

import math

import pytest

import paper_1109_1264_b200 as lv
from paper_1109_1264_b200 import benchmark as sb
from paper_1109_1264_b200.expressions import AssignNode, AssignReduceNode, ScaleNode, SumNode, as_node


def hv(n, dt="f64"):
    return lv.DenseVector.zeros(n, dt, device="cpu")


def test_accounting_matches_reference_for_shared_ops():
    # reference bench.py:9-15: dot 2s, scal 2s, axpy 3s, scaled_copy 2s
    assert [sb.bytes_moved(op, 10, "f32") for op in sb.OPS] == [80, 80, 120, 80]
    assert [sb.flop_count(op, 10) for op in sb.OPS] == [20, 10, 20, 10]
    assert sb.bytes_moved("t2", 2**28, "f64") == 8 * 2**30
    assert sb.bytes_moved("etree", 2**30, "f32") == 20 * 2**30


def test_csv_round_trip_and_header(tmp_path):
    recs = [sb.BenchRecord("dot", "engine", "f32", 64, 3, 1e-6, 2e-6, 0.128, 0.512),
            sb.BenchRecord("t2", "torch", "f64", 1024, 3, 2e-6, 3e-6, 2.048, 16.384, 0.0025, "B200", 1,
                           32768, 0.002048)]
    p = tmp_path / "a.csv"
    sb.emit_csv(recs[:1], str(p))
    lines = p.read_text().splitlines()
    assert lines[0] == "op,variant,type,n,reps,best_s,median_s,gflops,gbytes"
    assert sb.parse_csv(p.read_text())[0] == recs[0]
    sb.emit_csv(recs, str(p), extended=True)
    back = sb.parse_csv(p.read_text())
    assert back[1].pct_hbm == recs[1].pct_hbm and back[1].device == "B200"
    assert back[1] == recs[1]
    assert p.read_text().splitlines()[0].endswith(",pct_hbm,device,gpus,bytes,pct_hbm_nominal")
    with pytest.raises(ValueError):
        sb.parse_csv("bad,header\n")


@pytest.mark.parametrize("argv", [["--op", "nope"], ["--variants", "bogus"], ["--sizes", "x"],
                                  ["--reps", "0"], ["--sizes", "-4"]])
def test_cli_rejects_bad_usage_with_exit_2(argv):
    with pytest.raises(SystemExit) as e:
        sb.main(argv)
    assert e.value.code == 2


def test_reference_bench_surface():
    """The reference bench module's public names keep their meaning:
    simd_available (bench.py:92-94), record_lines (:222-231), the `naive`
    variant and the `packages` option (:135-141, :195-213)."""
    assert sb.simd_available("f32") is True and sb.simd_available("f64") is True
    assert list(sb.record_lines([])) == ["op,variant,type,n,reps,best_s,median_s,gflops,gbytes"]
    assert "naive" in sb.VARIANTS
    import inspect
    params = list(inspect.signature(sb.run_sweep).parameters)
    assert params[:8] == ["ops", "variants", "sizes", "dtype", "reps", "warmup", "seed", "packages"]
    params = list(inspect.signature(sb.measure).parameters)
    assert params[:8] == ["op", "variant", "n", "dtype", "reps", "warmup", "seed", "packages"]


def test_static_traffic_counter():
    a, b, c, d = hv(100), hv(100), hv(100), hv(100)
    t = lv.traffic(AssignNode(as_node(d), as_node(a) + (as_node(b) - as_node(c))))
    assert (t["vectors_read"], t["vectors_written"], t["bytes"]) == (3, 1, 3200)
    # the same leaf twice is loaded once; dest aliasing a leaf counts as a read
    assert lv.traffic(AssignNode(as_node(a), as_node(a) + ScaleNode(2.0, as_node(b))))["bytes"] == 2400
    assert lv.traffic(SumNode(as_node(a) * as_node(a)))["bytes"] == 800
    fused = AssignReduceNode(AssignNode(as_node(b), as_node(b) + ScaleNode(0.5, as_node(a))),
                             SumNode(as_node(b) * as_node(c)))
    assert lv.traffic(fused)["bytes"] == 8 * 100 * 4  # x, y, z read once, y written once
    e = lv.traffic(AssignNode(as_node(d), 2.0 * (as_node(a) + as_node(b)) - 3.0 * (as_node(c) - as_node(d))
                              + 0.5 * as_node(a)))
    assert e["vectors_read"] == 4 and e["vectors_written"] == 1


@pytest.mark.gpu
def test_small_gpu_sweep(tmp_path):
    recs = sb.run_sweep(["dot", "t2", "axpy_dot"], ["engine", "torch", "engine-U8"], [1000, 4097],
                        dtype="f64", reps=3, warmup=1)
    assert len(recs) == 3 * 3 * 2
    for r in recs:
        assert r.best_s > 0 and r.median_s >= r.best_s
        assert math.isclose(r.gbytes, sb.bytes_moved(r.op, r.n, r.type) / r.best_s / 1e9)
    host = sb.run_sweep(["t2", "dot"], ["engine-host"], [1 << 20], dtype="f32", reps=2, warmup=1)
    assert len(host) == 2
