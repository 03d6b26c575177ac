"""SM partition policy for colocated decode jobs (host logic, CPU)."""
import paper_2404_02015_b200 as mux


def test_byte_share_cfg2():
    s7, s13 = mux.spec("7b"), mux.spec("13b")
    ctx = [128 * 330, 128 * 330]
    sms = mux.byte_share_partitions([s7, s13], ctx, 148)
    assert sms == [56, 88]
    assert all(x % 8 == 0 for x in sms) and sum(sms) <= 148


def test_byte_share_is_proportional_and_whole_granules():
    specs = [mux.spec(m) for m in ("7b", "7b", "13b", "13b")]
    sms = mux.byte_share_partitions(specs, [0, 0, 0, 0], 148)
    assert sum(sms) == 144 and all(x % 8 == 0 and x >= 8 for x in sms)
    assert sms[0] == sms[1] and sms[2] == sms[3] and sms[2] > sms[0]


def test_byte_share_floor_one_granule():
    specs = [mux.spec("tiny-a"), mux.spec("13b")]
    sms = mux.byte_share_partitions(specs, [1, 10**6], 148)
    assert sms[0] == 8 and sum(sms) == 144
