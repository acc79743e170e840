"""Host-side pieces of SURVEY.md §8(f) against reference goldens (no GPU needed):
payload_upper_bound (planner.py:33-64), the DeviceTimeModel tables and lookups
(profiles.py:184-254, planner.py:67-75), and CLI argument errors that are raised before any
device work (cli.py:46-58 exit codes).  Goldens: tests/golden/make_cli_golden.py."""

import json
import os

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def host():
    with open(os.path.join(HERE, "golden", "host.json")) as f:
        return json.load(f)


def test_payload_upper_bound_matches_reference(host):
    import paper_2511_11608_b200 as sif

    for rec in host["bounds"]:
        kw = dict(rec["cfg"])
        if "fixed_q" in kw:
            kw["fixed_q"] = tuple(kw["fixed_q"])
        cfg = sif.CodecConfig(**kw)
        assert sif.payload_upper_bound(tuple(rec["shape"]), cfg) == rec["bits"], rec
        assert sif.payload_upper_bound(tuple(rec["shape"]), cfg, tuple(rec["split"])) == rec["bits_split"], rec
    with pytest.raises(sif.ConfigError):
        sif.payload_upper_bound((4, 4), sif.CodecConfig(s=0.5), (1, 1))


def test_max_payload_bytes_dominates_upper_bound(host):
    """The capacity used for output buffers is never below the reference's bound (and is
    above it where the reference bound is unsound: fixed q > q_bit)."""
    import paper_2511_11608_b200 as sif

    for rec in host["bounds"]:
        kw = dict(rec["cfg"])
        if "fixed_q" in kw:
            kw["fixed_q"] = tuple(kw["fixed_q"])
        cfg = sif.CodecConfig(**kw)
        r, c = rec["shape"]
        assert 8 * sif.max_payload_bytes(r, c, cfg) >= rec["bits"], rec


def test_time_model_lookups_match_reference(host, tmp_path):
    from paper_2511_11608_b200 import CodecConfig, DeviceTimeModel

    tm = host["timemodel"]
    m = DeviceTimeModel.from_dict(tm["table"])
    for L in tm["lookups"]:
        assert m.atkf_ms(L["s"], L["lam"]) == L["atkf"]
        assert m.ms_ms(L["m_plus"], L["m_minus"]) == L["ms"]
        assert m.abq_ms(L["q"]) == L["abq"]
        cfg = CodecConfig(s=L["s"], lam=L["lam"], m_plus=L["m_plus"], m_minus=L["m_minus"], q_bit=L["q"])
        assert m.encode_time_estimate(cfg) == L["est"]
    assert m.buffer_bytes(8000) == tm["buffer"]
    p = tmp_path / "tm.json"
    m.save(p)
    m2 = DeviceTimeModel.load(p)
    assert m2.t_atkf == m.t_atkf and m2.t_ms == m.t_ms and m2.t_abq == m.t_abq


@pytest.mark.parametrize("args,msg", [
    (["-s", "0.5", "--blocks", "3"], "error: --blocks expects 'M+,M-'"),
    (["-s", "1.5"], "error: s must be in [0, 1], got 1.5"),
    (["-s", "0.5", "--fixed-q", "8,x"], "error: bad Q list '8,x'; expected comma-separated integers"),
    (["-s", "0.5", "--blocks", "2,1", "--fixed-q", "6,3"],
     "error: Q vector of length 2 fits neither 2+1 nor a per-plane broadcast"),
])
def test_cli_config_errors(tmp_path, args, msg):
    from click.testing import CliRunner

    from paper_2511_11608_b200.cli import main

    src = tmp_path / "x.tns"
    src.write_bytes(b"TNS1")
    r = CliRunner(mix_stderr=False).invoke(main, ["encode", "--in", str(src), "--out", str(tmp_path / "o.sif")] + args)
    assert r.exit_code == 2
    assert r.stderr.splitlines()[0] == msg
