"""CPU: the CLI glue's argument handling (no device needed)."""
from paper_1111_6549_b200 import tool


def test_bench_refuses_runs_over_the_memory_budget(capsys):
    # gf2tool.cpp:314-322 -> exit 1 before any work (test_io_cli.cpp:372-374)
    assert tool.main(["bench", "--suite", "table1", "--sizes", "4096", "--memory-budget", "1000"]) == 1
    assert "memory-budget" in capsys.readouterr().err


def test_bench_rejects_unknown_suites_and_bad_k():
    assert tool.main(["bench", "--suite", "breakfast"]) == 1  # test_io_cli.cpp:210
    assert tool.main(["bench", "--suite", "table1", "--k", "0"]) == 1
    assert tool.main(["bench", "--suite", "table1", "--tables", "3"]) == 1


def test_check_budget_formula():
    tool.check_budget(64, 4 * 8 * 64)
    try:
        tool.check_budget(65, 4 * 8 * 65)
    except tool.BudgetError:
        pass
    else:
        raise AssertionError("65 columns need two words per row")
