"""GPU-aware AIO configuration (qk_config_tune): the chosen
Config keeps the reference's file format, and the Program the reference's own
optimizer (quokka_ref::aioOptimize) produces under it is byte-identical to
this framework's -- the tuner only picks knobs, it never changes the format
or the optimizer.  Host only."""
import pytest

from oracle import config_text


@pytest.mark.parametrize("kind,n,r,a,seed", [("qft", 24, 0, 0, 0), ("qaoa", 22, 0, 1, 3), ("bvones", 22, 0, 0, 0),
                                              ("qft", 26, 2, 0, 0), ("random", 24, 1, 200, 5)])
def test_tuned_config_pins_to_reference_optimizer(ref, qk, kind, n, r, a, seed):
    circ = qk.generate(kind, n, a, seed)
    cfg, report = qk.Config.tune(circ, n, r)
    assert "chosen:" in report and report.count("sweeps") == 12
    assert cfg.total_qubits == n and cfg.rank_qubits == r
    assert cfg.chunk_qubits in (12, 13) and cfg.buffer_qubits >= r
    # this engine fuses in its own passes: the reference's U5 / D_k fusion never wins
    assert cfg.fusion == 0 or cfg.fusion_qubits <= 4
    ini = cfg.text()
    assert ini == ref.config_roundtrip(ini)  # the reference parses and re-serializes it unchanged
    mine = qk.Program.optimize(circ, cfg).text()
    assert mine == ref.optimize(ref.circuit_roundtrip(circ), ini)


def test_buffer_sized_to_hbm_headroom(qk):
    circ = qk.generate("qft", 33)
    big, _ = qk.Config.tune(circ, 33, 0, 180e9)   # 128 GiB slice: ~41 GB left, 2 x 2^B x 16 B must fit
    small, _ = qk.Config.tune(circ, 33, 0, 150e9)
    assert big.buffer_qubits == 30 and small.buffer_qubits < big.buffer_qubits
