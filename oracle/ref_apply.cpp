// ref_apply.cpp -- TEST INFRASTRUCTURE ONLY. The reference CLI's `apply` subcommand restated over
// the UNMODIFIED reference headers (the CLI itself needs CLI11, which is absent): same file
// formats, same per-block float / fixed transforms, same exit codes. Used to produce the expected
// output files that paper_2505_21728_b200/hygt_gpu_apply is checked against.
//   reference: tools/hygt_main.cpp:130-172 (run_apply), :275-284 (exit codes)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hygt/bundle.hpp"
#include "hygt/dataset.hpp"
#include "hygt/fixedpoint.hpp"
#include "hygt/transform.hpp"

static int apply(const std::string& model, const std::string& data, bool forward, bool fixed,
                 const std::string& out) {
  const hygt::ModelBundle bundle = hygt::read_bundle(model);
  const hygt::ResidualDataset ds = hygt::read_rblk(data);
  if (ds.log2_n() != bundle.log2_n()) throw hygt::ArgumentError("apply: model/data dimension mismatch");
  if (ds.class_count() != bundle.class_count()) throw hygt::ArgumentError("apply: model/data class count mismatch");
  std::vector<hygt::ResidualBlock> result;
  result.reserve(ds.blocks().size());
  if (!fixed) {
    std::vector<hygt::HyGTModel> per_class;
    for (std::size_t c = 0; c < bundle.class_count(); ++c) per_class.push_back(bundle.dequantized(c));
    for (const hygt::ResidualBlock& blk : ds.blocks()) {
      const hygt::HyGTModel& m = per_class[blk.class_id];
      result.push_back({blk.class_id, forward ? hygt::forward(m, blk.values) : hygt::inverse(m, blk.values)});
    }
  } else {
    if (!bundle.quantized()) throw hygt::ArgumentError("apply: fixed arithmetic needs a quantized bundle");
    const hygt::TrigTable table(bundle.angle_bits(), bundle.precision_bits());
    for (const hygt::ResidualBlock& blk : ds.blocks()) {
      std::vector<std::int64_t> v(blk.values.size());
      for (std::size_t i = 0; i < v.size(); ++i) v[i] = std::llround(blk.values[i]);
      const hygt::QuantizedHyGTModel& m = bundle.quantized_model(blk.class_id);
      const std::vector<std::int64_t> y =
          forward ? hygt::forward_fixed(m, table, std::move(v)) : hygt::inverse_fixed(m, table, std::move(v));
      result.push_back({blk.class_id, std::vector<double>(y.begin(), y.end())});
    }
  }
  hygt::write_rblk(out, hygt::ResidualDataset(ds.log2_n(), ds.class_count(), std::move(result)));
  return 0;
}

int main(int argc, char** argv) {
  std::string model, data, out, direction = "forward", arithmetic = "float";
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i], v = argv[i + 1];
    if (k == "--model") model = v;
    else if (k == "--data") data = v;
    else if (k == "--out") out = v;
    else if (k == "--direction") direction = v;
    else if (k == "--arithmetic") arithmetic = v;
  }
  try {
    return apply(model, data, direction == "forward", arithmetic == "fixed", out);
  } catch (const hygt::ArgumentError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  } catch (const hygt::IoError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  } catch (const hygt::NumericalError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
