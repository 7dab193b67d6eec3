// DSPR front-end robustness against the device center — this repo's restatement of the
// reference's release-gate check 8 (acceptance.cpp:436-545): 1,000 malformed frames in
// five classes (bad magic, bad version, truncated payload, dim mismatch, NaN/Inf), each
// answered with its documented ERROR code; unparseable frames close the connection,
// recoverable ones keep it; the center is bit-for-bit untouched and counts 0 exchanges.
// Built by tests/cpp/Makefile against libdeepspark_b200.so; run by tests/test_dspr.py.
#include <bit>
#include <cstring>
#include <limits>
#include <map>
#include <string>

#include "deepspark/client.hpp"
#include "deepspark/exchanger.hpp"
#include "deepspark/net.hpp"
#include "deepspark/protocol.hpp"
#include "deepspark/rng.hpp"
#include "doctest.h"

using namespace deepspark;

namespace {

bool same_bits(const ParamVector& a, const ParamVector& b) {
  return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), 4 * a.size()) == 0);
}

ExchangerConfig fuzz_config() {
  ExchangerConfig cfg;
  cfg.bind_address = "127.0.0.1:0";
  cfg.pool_size = 2;
  cfg.alpha = 0.1f;
  cfg.model = Model::softmax(4, 3);  // dim 15
  cfg.init_seed = 9;
  return cfg;
}

}  // namespace

TEST_SUITE("dspr") {

TEST_CASE("1000 malformed frames draw their ERROR codes and leave the center untouched") {
  ExchangerService svc(fuzz_config());
  const ParamVector initial = svc.master().snapshot();
  const HostPort addr{"127.0.0.1", svc.port()};
  const uint32_t dim = static_cast<uint32_t>(initial.size());
  REQUIRE(dim == 15);
  Rng rng(42);
  std::map<uint16_t, int> seen;
  int failures = 0;
  for (int k = 0; k < 1000 && failures == 0; ++k) {
    ParamVector good(dim);
    for (auto& x : good) x = static_cast<float>(rng.normal());
    std::vector<uint8_t> frame;
    uint16_t want = 0;
    bool closes = false;
    switch (k % 5) {
      case 0:  // one corrupted magic byte
        frame = wire::encode_frame(wire::kExchangeReq, wire::build_params(good));
        frame[rng.below(4)] ^= static_cast<uint8_t>(1 + rng.below(255));
        want = wire::kErrBadFrame, closes = true;
        break;
      case 1:  // unsupported version
        frame = wire::encode_frame(wire::kExchangeReq, wire::build_params(good));
        frame[4] = static_cast<uint8_t>(2 + rng.below(200));
        want = wire::kErrBadFrame, closes = true;
        break;
      case 2: {  // payload shorter than its declared dim
        auto p = wire::build_params(good);
        p.resize(p.size() - 4 * (1 + rng.below(4)));
        frame = wire::encode_frame(wire::kExchangeReq, p);
        want = wire::kErrBadFrame, closes = true;
        break;
      }
      case 3: {  // well-formed vector of the wrong size
        ParamVector small(1 + rng.below(dim - 1));
        for (auto& x : small) x = static_cast<float>(rng.normal());
        frame = wire::encode_frame(wire::kExchangeReq, wire::build_params(small));
        want = wire::kErrDimMismatch;
        break;
      }
      default:  // NaN or Inf in the payload
        good[rng.below(dim)] =
            (k % 2) ? std::numeric_limits<float>::quiet_NaN() : std::numeric_limits<float>::infinity();
        frame = wire::encode_frame(wire::kExchangeReq, wire::build_params(good));
        want = wire::kErrNonFinite;
        break;
    }
    Socket sock = tcp_connect(addr, 5000);
    sock.set_timeouts(5000, 5000);
    sock.send_all(frame.data(), frame.size());
    const auto reply = read_frame(sock);
    if (!reply || reply->msg_type != wire::kError) {
      ++failures;
      CAPTURE(k);
      CHECK(false);
      break;
    }
    const wire::ErrorMsg err = wire::parse_error(reply->payload);
    ++seen[err.code];
    if (err.code != want) {
      ++failures;
      CAPTURE(k);
      CHECK(err.code == want);
    }
    if (closes) {
      if (read_frame(sock).has_value()) ++failures, CHECK(false);  // must hang up after a bad frame
    } else if (k % 50 == 0) {  // a recoverable error keeps the dialogue alive
      write_frame(sock, wire::kStatsReq, {});
      const auto stats = read_frame(sock);
      CHECK((stats && stats->msg_type == wire::kStatsResp));
    }
    sock.close();
    if (k % 100 == 99) CHECK(same_bits(svc.master().snapshot(), initial));
  }
  CHECK(failures == 0);
  CHECK(seen[wire::kErrBadFrame] == 600);
  CHECK(seen[wire::kErrDimMismatch] == 200);
  CHECK(seen[wire::kErrNonFinite] == 200);
  CHECK(same_bits(svc.master().snapshot(), initial));
  CHECK(svc.master().exchange_count() == 0);
  svc.stop();
}

TEST_CASE("a reference-speaking client trains against the GPU center over TCP") {
  // EXCHANGE_REQ round trips equal the device elastic kernel applied in order
  ExchangerService svc(fuzz_config());
  ExchangerClient c(HostPort{"127.0.0.1", svc.port()});
  const wire::ConfigMsg cfg = c.hello();
  CHECK(cfg.param_dim == 15);
  CHECK(cfg.model_fingerprint == Model::softmax(4, 3).fingerprint());
  ParamVector m = c.fetch_initial();
  Rng rng(5);
  for (int r = 0; r < 20; ++r) {
    ParamVector w(15);
    for (auto& x : w) x = static_cast<float>(rng.normal());
    const ParamVector got = c.exchange(w);
    for (size_t i = 0; i < w.size(); ++i) {
      float wo, mo;
      elastic_update_elem(w[i], m[i], 0.1f, wo, mo);
      CHECK(std::bit_cast<uint32_t>(got[i]) == std::bit_cast<uint32_t>(wo));
      m[i] = mo;
    }
  }
  CHECK(same_bits(svc.master().snapshot(), m));
  CHECK(c.stats().exchange_count == 20);
  svc.stop();
}

}  // TEST_SUITE
