// Self-test of tests/cpp/doctest_shim/doctest.h: SUBCASE pass structure
// (one leaf per pass, nesting, code outside subcases every pass), failure
// accounting, REQUIRE aborting a pass, exception macros, Approx.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <stdexcept>
#include <string>

static std::string trace;

TEST_CASE("subcases: leaves run once each, prefix every pass") {
  trace += "P";
  SUBCASE("a") { trace += "a"; }
  SUBCASE("b") {
    trace += "b";
    SUBCASE("b1") { trace += "1"; }
    SUBCASE("b2") { trace += "2"; }
  }
  SUBCASE("c") { trace += "c"; }
  trace += ".";
}

TEST_CASE("trace check") {
  // passes: P a . | P b 1 . | P b 2 . | P c .
  CHECK(trace == "Pa.Pb1.Pb2.Pc.");
}

TEST_CASE("expected failures (4 failed assertions, REQUIRE ends the pass)") {
  CHECK(1 == 2);
  CHECK_FALSE(true);
  CHECK_THROWS_AS(throw std::runtime_error("x"), std::invalid_argument);
  CHECK_THROWS_AS(throw std::invalid_argument("x"), std::invalid_argument);
  CHECK_THROWS_WITH_AS(throw std::invalid_argument("msg"), "msg", std::invalid_argument);
  CHECK_THROWS(throw 1);
  CHECK(0.1 + 0.2 == doctest::Approx(0.3));
  CHECK(1.0 != doctest::Approx(1.1));
  REQUIRE(false);
  CHECK(false);  // not reached: REQUIRE aborted the pass
}

TEST_CASE("unexpected exception") { throw std::logic_error("boom"); }
