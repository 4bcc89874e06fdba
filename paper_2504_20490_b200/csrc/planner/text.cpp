// hshard-b200 planner: text forms.
//
// * parse_annotation: inverse of HetAnnotation::str() (annotation.cpp:146-170
//   in the reference), the wire format of the C ABI.
// * dump_plan / dump_bsr / dump_table: the canonical JSON used for byte-exact
//   plan parity against the reference planner (oracle/ref_tool.cpp emits the
//   same format from the reference's own objects).
#include <cctype>
#include <sstream>

#include "hshard/resolve.hpp"

namespace hshard {

namespace {

class Cursor {
 public:
  explicit Cursor(const std::string& s) : s_(s) {}
  void skip_ws() {
    while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
  }
  bool eat(char c) {
    skip_ws();
    if (i_ < s_.size() && s_[i_] == c) {
      ++i_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) bad(std::string("expected '") + c + "'");
  }
  bool eat_word(const char* w) {
    skip_ws();
    const std::string word(w);
    if (s_.compare(i_, word.size(), word) == 0) {
      i_ += word.size();
      return true;
    }
    return false;
  }
  int64_t integer() {
    skip_ws();
    size_t j = i_;
    if (j < s_.size() && (s_[j] == '-' || s_[j] == '+')) ++j;
    const size_t digits = j;
    while (j < s_.size() && std::isdigit(static_cast<unsigned char>(s_[j]))) ++j;
    if (j == digits) bad("expected integer");
    const int64_t v = std::stoll(s_.substr(i_, j - i_));
    i_ = j;
    return v;
  }
  std::string until_end() {
    skip_ws();
    std::string r = s_.substr(i_);
    i_ = s_.size();
    return r;
  }
  bool done() {
    skip_ws();
    return i_ >= s_.size();
  }
  [[noreturn]] void bad(const std::string& why) const {
    fail(Errc::ParseError, why + " at offset " + std::to_string(i_) + " in '" + s_ + "'");
  }

 private:
  const std::string& s_;
  size_t i_ = 0;
};

ShardSpec read_spec(Cursor& c) {
  ShardSpec ds;
  c.expect('{');
  if (c.eat('}')) return ds;
  do {
    const int key = static_cast<int>(c.integer());
    c.expect(':');
    ds.entries.push_back({key, static_cast<int>(c.integer())});
  } while (c.eat(','));
  c.expect('}');
  return ds;
}

}  // namespace

ShardSpec parse_shard_spec(const std::string& text) {
  Cursor c(text);
  ShardSpec ds = read_spec(c);
  if (!c.done()) c.bad("trailing text");
  return ds;
}

HetAnnotation parse_annotation(const std::string& text) {
  Cursor c(text);
  if (c.eat_word("hsize=")) c.integer();  // implied by the group count
  if (!c.eat_word("hdim=")) c.bad("expected hdim=");
  const int hdim = static_cast<int>(c.integer());
  std::vector<DeviceGroup> groups;
  std::vector<ShardSpec> specs;
  c.expect('[');
  do {
    c.expect('(');
    std::vector<DeviceId> devs;
    if (!c.eat(')')) {
      do devs.push_back(static_cast<DeviceId>(c.integer()));
      while (c.eat(','));
      c.expect(')');
    }
    groups.emplace_back(std::move(devs));
    specs.push_back(read_spec(c));
  } while (c.eat(';'));
  c.expect(']');
  std::vector<Rational> ratios;
  if (c.eat_word("ratios=")) {
    std::stringstream ss(c.until_end());
    std::string tok;
    while (std::getline(ss, tok, ','))
      if (!tok.empty()) ratios.push_back(Rational::parse(tok));
  }
  if (!c.done()) c.bad("trailing text");
  return HetAnnotation::make(std::move(groups), std::move(specs), hdim, std::move(ratios));
}

Bandwidth parse_bandwidth(const std::string& text) {
  Bandwidth bw = Bandwidth::uniform();
  std::stringstream ss(text);
  std::string item;
  while (std::getline(ss, item, ';')) {
    size_t a = item.find_first_not_of(' '), b = item.find_last_not_of(' ');
    if (a == std::string::npos) continue;
    item = item.substr(a, b - a + 1);
    if (item == "u") continue;
    const size_t eq = item.find('=');
    if (eq == std::string::npos) fail(Errc::ParseError, "bad bandwidth item '" + item + "'");
    const std::string key = item.substr(0, eq);
    const double w = std::stod(item.substr(eq + 1));
    if (key == "d") {
      bw.default_bw = w;
      continue;
    }
    const size_t dash = key.find('-', 1);
    if (dash == std::string::npos) fail(Errc::ParseError, "bad bandwidth link '" + key + "'");
    bw.set(std::stoi(key.substr(0, dash)), std::stoi(key.substr(dash + 1)), w);
  }
  return bw;
}

// ---------------------------------------------------------------- dumps
namespace {

struct Json {
  std::string out;

  Json& raw(const std::string& s) {
    out += s;
    return *this;
  }
  Json& num(int64_t v) { return raw(std::to_string(v)); }
  Json& str(const std::string& s) {
    out += '"';
    for (char ch : s) {
      if (ch == '"' || ch == '\\') out += '\\';
      out += ch;
    }
    out += '"';
    return *this;
  }
  template <class Seq>
  Json& ints(const Seq& v) {
    out += '[';
    bool first = true;
    for (auto x : v) {
      if (!first) out += ',';
      first = false;
      out += std::to_string(x);
    }
    out += ']';
    return *this;
  }
  Json& region(const SliceRegion& r) {
    const bool ordinals = r.partial_index != 0 || r.partial_count != 1 || r.replica_index != 0 ||
                          r.replica_count != 1;
    if (ordinals) raw("{\"b\":");
    out += '[';
    for (size_t d = 0; d < r.bounds.size(); ++d) {
      if (d) out += ',';
      raw("[").num(r.bounds[d][0]).raw(",").num(r.bounds[d][1]).raw("]");
    }
    out += ']';
    if (ordinals)
      raw(",\"p\":[").num(r.partial_index).raw(",").num(r.partial_count).raw("],\"q\":[")
          .num(r.replica_index).raw(",").num(r.replica_count).raw("]}");
    return *this;
  }
  template <class Seq, class Fn>
  Json& list(const Seq& seq, Fn&& each) {
    out += '[';
    bool first = true;
    for (const auto& x : seq) {
      if (!first) out += ',';
      first = false;
      each(x);
    }
    out += ']';
    return *this;
  }
};

void bsr_into(Json& j, const BsrPlan& p) {
  j.raw("{\"local\":").list(p.local_copies, [&](const LocalCopy& c) {
    j.raw("[").num(c.device).raw(",").num(c.tensor_id).raw(",").region(c.region).raw("]");
  });
  j.raw(",\"xfer\":").list(p.transfers, [&](const Transfer& t) {
    j.raw("[").num(t.tensor_id).raw(",").region(t.region).raw(",").num(t.sender).raw(",")
        .num(t.receiver).raw(",").num(t.bytes).raw("]");
  });
  j.raw(",\"fg\":").list(p.fusion_groups, [&](const FusionGroup& g) {
    j.raw("[").num(g.sender).raw(",").num(g.receiver).raw(",").ints(g.transfer_indices).raw("]");
  });
  j.raw("}");
}

void step_into(Json& j, const CommStep& s) {
  j.raw("{\"kind\":").str(step_kind_name(s.kind)).raw(",\"sub\":").num(s.subgroup);
  j.raw(",\"groups\":").list(s.groups, [&](const std::vector<DeviceId>& g) { j.ints(g); });
  j.raw(",\"pairs\":").list(s.pairs, [&](const std::pair<DeviceId, DeviceId>& p) {
    j.raw("[").num(p.first).raw(",").num(p.second).raw("]");
  });
  j.raw(",\"slices\":").list(s.slices, [&](const SliceCollective& sc) {
    j.raw("{\"reg\":").region(sc.region).raw(",\"c\":").ints(sc.contributors).raw(",\"r\":")
        .ints(sc.receivers).raw("}");
  });
  j.raw(",\"bsr\":");
  if (s.bsr)
    bsr_into(j, *s.bsr);
  else
    j.raw("null");
  j.raw("}");
}

}  // namespace

std::string dump_bsr(const BsrPlan& plan) {
  Json j;
  bsr_into(j, plan);
  return j.out;
}

std::string dump_table(const BsrTable& table) {
  Json j;
  j.raw("{\"rows\":").list(table.rows, [&](const BsrRow& r) {
    j.raw("[").num(r.tensor_id).raw(",").region(r.region).raw(",").ints(r.owners).raw(",")
        .ints(r.requesters).raw(",").num(r.bytes).raw("]");
  });
  j.raw("}");
  return j.out;
}

std::string dump_plan(const CommPlan& p) {
  Json j;
  j.raw("{\"src\":").str(p.src.str()).raw(",\"dst\":").str(p.dst.str()).raw(",\"mid\":");
  if (p.mid)
    j.str(p.mid->str());
  else
    j.raw("null");
  j.raw(",\"shape\":").ints(p.shape).raw(",\"dtype\":").str(dtype_name(p.dtype));
  j.raw(",\"bottom\":").list(p.bottom_phase, [&](const CommStep& s) { step_into(j, s); });
  j.raw(",\"top\":").list(p.top_phase, [&](const CommStep& s) { step_into(j, s); });
  j.raw("}");
  return j.out;
}

}  // namespace hshard
