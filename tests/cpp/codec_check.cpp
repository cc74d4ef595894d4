// TEST INFRASTRUCTURE — the JSONL codec of the collector, exercised without a
// GPU: built once against the reference's collector.cpp (codec_ref) and once
// against the B200 drop-in library (codec_b200); tests/test_collector_codec.py
// requires identical output. Prints the encoded records of deterministic
// pseudo-random metas / spans (integers, negative tags, doubles over the whole
// exponent range, escapes, UTF-8), then the outcome of parsing tricky lines
// (system specs, and ingest() of streams that fail before any GPU step).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <iostream>
#include <string>
#include <vector>

#include "strata/collector.hpp"

using namespace strata;

static std::uint64_t s = 0x9E3779B97F4A7C15ull;
static std::uint64_t rnd() {
  std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static double rnd_double() {
  switch (rnd() % 6) {
    case 0: { double d; std::uint64_t b = rnd(); std::memcpy(&d, &b, 8); return std::isfinite(d) ? d : 1.5; }
    case 1: return static_cast<double>(rnd() % 100000) / 1000.0;
    case 2: return static_cast<double>(rnd() % 1000) * std::pow(10.0, static_cast<int>(rnd() % 40) - 20);
    case 3: return static_cast<double>(rnd() % 1000000);
    case 4: return std::ldexp(static_cast<double>(rnd() % (1ull << 53)), static_cast<int>(rnd() % 200) - 100);
    default: return (rnd() & 1) ? 0.0 : -0.0;
  }
}

static std::string rnd_string() {
  static const char* pieces[] = {"conv", "\"q\"", "back\\slash", "tab\t", "nl\n", "\x01\x1f", "caf\xc3\xa9",
                                 "\xe2\x82\xac", "\xf0\x9f\x98\x80", "/", " ", "sgemm_128x64"};
  std::string out;
  for (int k = 0, n = 1 + rnd() % 3; k < n; ++k) out += pieces[rnd() % 12];
  return out;
}

int main() {
  for (int i = 0; i < 300; ++i) {
    RunMeta m;
    m.trace_id = rnd();
    m.batch_size = static_cast<std::uint32_t>(rnd());
    m.run_index = static_cast<std::uint32_t>(rnd() % 100);
    for (int l = 0; l < 4; ++l)
      if (rnd() & 1) m.profiling_levels.insert(static_cast<Level>(l));
    m.serialized = rnd() & 1;
    m.system = SystemSpec{rnd_string(), rnd_double(), rnd_double()};
    std::cout << encode_meta_record(m) << "\n";
    std::cout << encode_system_spec(m.system) << "\n";
    Span sp;
    sp.trace_id = rnd();
    sp.span_id = rnd();
    if (rnd() & 1) sp.parent_id = rnd();
    if (rnd() & 1) sp.correlation_id = rnd() % 1000;
    sp.name = rnd_string();
    sp.level = static_cast<Level>(rnd() % 4);
    sp.kind = static_cast<SpanKind>(rnd() % 3);
    sp.begin_ns = rnd();
    sp.end_ns = rnd();
    for (int t = 0, n = rnd() % 5; t < n; ++t) {
      switch (rnd() % 3) {
        case 0: sp.tags[rnd_string()] = static_cast<std::int64_t>(rnd()); break;
        case 1: sp.tags[rnd_string()] = rnd_double(); break;
        default: sp.tags[rnd_string()] = rnd_string();
      }
    }
    std::cout << encode_span_record(sp) << "\n";
  }
  // doubles over every exponent (random bit patterns) and near powers of ten
  for (int i = 0; i < 200000; ++i) {
    double d;
    if (i % 2) {
      std::uint64_t b = rnd();
      std::memcpy(&d, &b, 8);
      if (!std::isfinite(d)) continue;
    } else {
      d = std::nextafter(std::pow(10.0, static_cast<int>(rnd() % 600) - 300), (rnd() & 1) ? 0.0 : 1e308);
    }
    std::cout << encode_system_spec(SystemSpec{"d", d, -d}) << "\n";
  }
  const char* specs[] = {
      "{\"name\":\"v100\",\"peak_flops\":15.7e12,\"mem_bw\":900e9}",
      "{\"name\":\"x\",\"peak_flops\":1,\"mem_bw\":-2}",
      "{\"name\":\"x\",\"peak_flops\":18446744073709551615,\"mem_bw\":184467440737095516160}",
      "{\"name\":\"\\u00e9\\ud83d\\ude00\",\"peak_flops\":1e400,\"mem_bw\":-9223372036854775808}",
      "{\"name\":\"dup\",\"name\":\"second\",\"peak_flops\":0.1,\"mem_bw\":2.5E-3}",
      " \t{\"name\":\"ws\" , \"peak_flops\" : 1.0 , \"mem_bw\" : 1 } \r",
      "{\"name\":\"x\"}", "{", "[]", "{\"name\":1,\"peak_flops\":1,\"mem_bw\":1}",
      "{\"name\":\"x\",\"peak_flops\":01,\"mem_bw\":1}", "{\"name\":\"x\",\"peak_flops\":1.,\"mem_bw\":1}",
      "{\"name\":\"x\",\"peak_flops\":\"1\",\"mem_bw\":1}", "{\"name\":\"\\x\",\"peak_flops\":1,\"mem_bw\":1}",
      "{\"name\":\"a\tb\",\"peak_flops\":1,\"mem_bw\":1}", "{\"name\":\"\\ud800\",\"peak_flops\":1,\"mem_bw\":1}",
      "{\"name\":\"\xc3\",\"peak_flops\":1,\"mem_bw\":1}", "{\"name\":\"x\",\"peak_flops\":1,\"mem_bw\":1} x",
      "{\"name\":\"x\",\"peak_flops\":-0,\"mem_bw\":-0.0}", "{\"name\":\"x\",\"peak_flops\":true,\"mem_bw\":1}",
  };
  for (const char* t : specs) {
    try {
      std::cout << "spec ok " << encode_system_spec(parse_system_spec(t)) << "\n";
    } catch (const IngestError& e) {
      std::cout << "spec IngestError " << e.what() << "\n";
    }
  }
  const std::string meta =
      "{\"rec\":\"meta\",\"trace_id\":7,\"batch_size\":1,\"run_index\":0,\"levels\":[\"model\",\"layer\"],"
      "\"system\":{\"name\":\"v\",\"peak_flops\":1,\"mem_bw\":1}}\n";
  const std::string span = "{\"rec\":\"span\",\"trace_id\":7,\"span_id\":1,\"name\":\"m\",\"level\":\"model\","
                           "\"kind\":\"sync\",\"begin_ns\":0,\"end_ns\":5";
  const std::vector<std::string> streams = {
      "", "\n  \n", "not json\n", meta + meta, span + "}\n",
      meta + "[1,2]\n", meta + span + ",\"tags\":[]}\n", meta + span + ",\"tags\":{\"a\":null}}\n",
      meta + span + ",\"parent_id\":-1}\n", meta + span + ",\"correlation_id\":1.5}\n",
      meta + "{\"rec\":\"span\",\"trace_id\":7,\"span_id\":1,\"name\":\"m\",\"level\":\"bogus\",\"kind\":\"sync\","
             "\"begin_ns\":0,\"end_ns\":5}\n",
      meta + "{\"rec\":\"span\",\"trace_id\":7,\"span_id\":1,\"name\":\"m\",\"level\":\"model\",\"kind\":\"x\","
             "\"begin_ns\":0,\"end_ns\":5}\n",
      meta + "{\"rec\":\"span\",\"trace_id\":7,\"span_id\":1,\"level\":\"model\",\"kind\":\"sync\","
             "\"begin_ns\":0,\"end_ns\":5}\n",
      meta + "{\"rec\":\"span\",\"trace_id\":8,\"span_id\":1,\"name\":\"m\",\"level\":\"model\",\"kind\":\"sync\","
             "\"begin_ns\":0,\"end_ns\":5}\n",
      "{\"rec\":\"meta\",\"trace_id\":7,\"batch_size\":1,\"run_index\":0,\"levels\":[\"model\",\"warp\"],"
      "\"system\":{\"name\":\"v\",\"peak_flops\":1,\"mem_bw\":1}}\n",
      "{\"rec\":\"meta\",\"trace_id\":7,\"batch_size\":1,\"run_index\":0,\"levels\":\"model\","
      "\"system\":{\"name\":\"v\",\"peak_flops\":1,\"mem_bw\":1}}\n",
      "{\"rec\":\"meta\",\"trace_id\":7,\"batch_size\":1,\"run_index\":0,\"levels\":[],\"serialized\":1,"
      "\"system\":{\"name\":\"v\",\"peak_flops\":1,\"mem_bw\":1}}\n",
      "{\"rec\":\"meta\",\"trace_id\":7,\"batch_size\":1,\"run_index\":0,\"levels\":[]}\n",
      "{\"rec\":\"meta\",\"trace_id\":7,\"batch_size\":1,\"run_index\":0,\"levels\":[],\"system\":3}\n",
      "{\"rec\":\"other\"}\n" + meta + "{\"rec\":\"span\",\"trace_id\":7,\"span_id\":1,\"name\":\"m\"}\n",
  };
  for (const std::string& t : streams) {
    try {
      ingest_string(t);
      std::cout << "ingest ok\n";
    } catch (const IngestError& e) {
      std::cout << "ingest IngestError " << e.what() << "\n";
    }
  }
  return 0;
}
