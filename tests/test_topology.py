"""Stage roles and hand-off routes for asymmetric plans (pure host logic)."""

import pytest

from paper_2311_11514_b200.config import LLAMA2_70B, TINY
from paper_2311_11514_b200.plan import GlobalAssignment, InputError, StageAssignment, simple_plan
from paper_2311_11514_b200.topology import pipeline_roles, role_of


def test_422_routes():
    roles = {r.device: r for r in pipeline_roles(simple_plan([4, 2, 2], [40, 20, 20]), 0, LLAMA2_70B)}
    # stage 0 (TP4) -> stage 1 (TP2): receiver r' pulls from sender r' mod 4
    assert roles[0].send_to == (4,) and roles[1].send_to == (5,)
    assert roles[2].send_to == () and roles[3].send_to == ()
    assert roles[4].recv_from == 0 and roles[5].recv_from == 1
    assert roles[6].recv_from == 4 and roles[7].recv_from == 5
    # tokens return from the last stage (TP2) to stage 0 (TP4): r' <- r' mod 2
    assert roles[6].ids_send_to == (0, 2) and roles[7].ids_send_to == (1, 3)
    assert [roles[d].ids_recv_from for d in range(4)] == [6, 7, 6, 7]
    assert roles[0].layers == (0, 40) and roles[7].layers == (60, 80)
    assert roles[5].tp_group == (4, 5) and roles[5].tp_rank == 1


def test_fan_out_when_next_stage_is_wider():
    roles = {r.device: r for r in pipeline_roles(simple_plan([1, 2, 1], [1, 2, 1]), 0, TINY)}
    assert roles[0].send_to == (1, 2)
    assert roles[1].send_to == (3,) and roles[2].send_to == ()
    assert roles[3].ids_send_to == (0,)


def test_every_receiver_gets_exactly_one_message():
    for tps in ([4, 2, 2], [2, 1], [1, 4, 2], [2, 2], [8]):
        roles = pipeline_roles(simple_plan(tps, [80 // len(tps)] * (len(tps) - 1) + [80 - 80 // len(tps) * (len(tps) - 1)]), 0, LLAMA2_70B)
        sent = [d for r in roles for d in r.send_to]
        recv = [r.device for r in roles if r.stage > 0]
        assert sorted(sent) == sorted(recv)


def test_validation():
    bad = GlobalAssignment(((StageAssignment((0, 1), 3), StageAssignment((2,), 2)),))
    with pytest.raises(ValueError):
        pipeline_roles(bad, 0, TINY)
    with pytest.raises(InputError):  # 8 heads not divisible by TP 3
        pipeline_roles(simple_plan([3], [4]), 0, TINY)
    p, r = role_of(simple_plan([2, 1], [3, 1]), 2, TINY)
    assert p == 0 and r.stage == 1 and r.is_last
    assert role_of(simple_plan([2, 1], [3, 1]), 5, TINY) == (None, None)
