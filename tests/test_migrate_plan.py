"""Host logic of expert migration (paper_2401_08383_b200/migrate.py): slot
rule and move plan between two placements."""
import numpy as np

from paper_2401_08383_b200 import migrate


def test_slot_table_expert_order():
    a = np.array([[0, 1, 0, 1], [1, 1, 0, 0]])
    assert migrate.slot_table(a, 2).tolist() == [[0, 0, 1, 1], [0, 1, 0, 1]]


def test_plan_identity_is_empty():
    a = np.array([[0, 0, 1, 1], [1, 0, 1, 0]])
    assert migrate.plan(a, a, 2) == []


def test_plan_moves_and_slot_shuffles():
    old = np.array([[0, 0, 1, 1]])
    new = np.array([[1, 0, 0, 1]])
    # expert 0: gpu0 slot0 -> gpu1 slot0; expert 1: gpu0 slot1 -> gpu0 slot0
    # (stays, new slot); expert 2: gpu1 slot0 -> gpu0 slot1; expert 3: gpu1
    # slot1 -> gpu1 slot1 (unchanged)
    assert migrate.plan(old, new, 2) == [(0, 0, 0, 0, 1, 0), (0, 1, 0, 1, 0, 0), (0, 2, 1, 0, 0, 1)]
