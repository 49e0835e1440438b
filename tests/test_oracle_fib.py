"""Pins for the fib oracle.

The oracle is a plain recursion. It is pinned here against computations that
are NOT that recursion:
  * an iterative Fibonacci loop (value),
  * the golden values the paper / SPEC / OEIS print (tests/golden/fib.txt),
  * closed forms for the call tree: calls = 2F(n+1)-1, invocations =
    3F(n+1)-2 (leaves run one state, internal calls two),
  * a brute-force simulation of the transformed state machine with an explicit
    work list and join counters (no recursion) for small n.
"""
import os

import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def fib_iter(n):
    a, b = 0, 1
    for _ in range(n):
        a, b = b, a + b
    return a


def read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                rows.append([int(t) for t in line.split()[:3] if t.lstrip("-").isdigit()])
    return rows


@pytest.mark.parametrize("n", range(0, 31))
def test_value_and_counts_closed_form(n):
    v, calls, inv = oracle.fib(n)
    assert v == fib_iter(n)
    assert calls == 2 * fib_iter(n + 1) - 1
    assert inv == 3 * fib_iter(n + 1) - 2


def test_golden_values():
    for n, val in read_golden("fib.txt"):
        if n <= 30:
            assert oracle.fib(n)[0] == val, n
        assert fib_iter(n) == val, n


def test_golden_task_counts():
    for n, tasks, inv in read_golden("fib_tasks.txt"):
        assert tasks == 2 * fib_iter(n + 1) - 1
        assert inv == 3 * fib_iter(n + 1) - 2
        if n <= 30:
            assert oracle.fib(n)[1:] == (tasks, inv)


@pytest.mark.slow
def test_fib40_full():
    v, calls, inv = oracle.fib(40)
    assert (v, calls, inv) == (102334155, 331160281, 496740421)


def simulate_state_machine(n0):
    """Sequential simulation of the transformed fib.

    Records carry {n, state, pending, parent, ordinal, res[2]}; a LIFO work
    list plays the runtime; case 0 of n >= 2 spawns two children and
    prepare_for_join(1); a finishing child stores into parent.res[ordinal]
    and decrements the parent's pending count; the parent is re-enqueued when
    it reaches 0 and resumes in case 1 with load_result(0) + load_result(1).
    """
    recs = [dict(n=n0, state=0, pending=0, parent=None, ordinal=0, res=[None, None])]
    work = [0]
    invocations = 0
    root_result = None
    while work:
        t = work.pop()
        r = recs[t]
        invocations += 1
        if r["state"] == 0 and r["n"] >= 2:
            for o, m in enumerate((r["n"] - 1, r["n"] - 2)):
                recs.append(dict(n=m, state=0, pending=0, parent=t, ordinal=o, res=[None, None]))
                work.append(len(recs) - 1)
            r["pending"] = 2
            r["state"] = 1
            continue
        if r["state"] == 0:
            result = r["n"]
        else:
            assert None not in r["res"], "continuation ran before its children finished"
            result = r["res"][0] + r["res"][1]
        r["state"] = -1  # finished
        p = r["parent"]
        if p is None:
            root_result = result
        else:
            recs[p]["res"][r["ordinal"]] = result
            recs[p]["pending"] -= 1
            if recs[p]["pending"] == 0:
                work.append(p)
    return root_result, len(recs), invocations


@pytest.mark.parametrize("n", [0, 1, 2, 3, 5, 10, 15])
def test_brute_force_state_machine(n):
    assert simulate_state_machine(n) == oracle.fib(n)


def test_fib3_join_loads():
    # after fib(3)'s join, load_result(0) = fib(2) = 1, load_result(1) = fib(1) = 1
    assert oracle.fib(2)[0] == 1 and oracle.fib(1)[0] == 1 and oracle.fib(3)[0] == 2


def test_range_checked():
    with pytest.raises(ValueError):
        oracle.fib(-1)


# ---- fib with cutoff (EPAQ benchmark) ----

def _fib_cut_tasks(n, c):
    """Task count by an explicit work list (no recursion): a task n >= max(c, 2) has two children."""
    tasks, work = 0, [n]
    while work:
        m = work.pop()
        tasks += 1
        if m >= c and m >= 2:
            work += [m - 1, m - 2]
    return tasks


@pytest.mark.parametrize("n", range(0, 25))
@pytest.mark.parametrize("c", [0, 1, 2, 3, 5, 10])
def test_fib_cutoff(n, c):
    v, tasks, inv, serial = oracle.fib_cutoff(n, c)
    assert v == fib_iter(n)
    assert tasks == _fib_cut_tasks(n, c)
    # every non-leaf task runs 2 invocations, every leaf 1
    internal = (tasks - 1) // 2
    assert inv == 2 * internal + (tasks - internal)
    # serial work: each cutoff task m does 2F(m+1)-1 serial calls of the naive recursion
    if c <= 2:
        assert (tasks, inv) == oracle.fib(n)[1:]  # cutoff <= 2 is the no-cutoff program


def test_fib_cutoff_serial_calls_closed_form():
    n, c = 20, 10
    _, tasks, _, serial = oracle.fib_cutoff(n, c)
    # leaves of the task tree are fib(9) and fib(8) tasks; count them by explicit expansion
    leaves = {}
    work = [n]
    while work:
        m = work.pop()
        if m >= c:
            work += [m - 1, m - 2]
        else:
            leaves[m] = leaves.get(m, 0) + 1
    assert serial == sum(k * (2 * fib_iter(m + 1) - 1) for m, k in leaves.items())
